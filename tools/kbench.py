"""Krylov-loop microbenchmark at a config: us per IOM2 iteration."""
import sys, time, ctypes as C
import numpy as np
sys.path.insert(0, ".")
from paper_1805_02144_b200.states import make_config
from paper_1805_02144_b200 import swe as gswe, _native as nat
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 40
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
lvl = None
if ":" in name:
    name, lvl = name.split(":")
ops, u0, spec = make_config(name, level=lvl)
ctx = gswe.SweContext(ops)
info = (C.c_int64 * 14)()
nat.check(nat.load().eik_swe_info(ctx.h, info))
print("info G,TPB,tiles,e1max,e2max,K,KC,tiled_ok,smem =", list(info))
v = np.random.default_rng(0).standard_normal(u0.shape[0])
if "f" in sys.argv[4:]:
    v = spec.dt * ctx.rhs(u0)
out = (C.c_double * 2)()
u = np.ascontiguousarray(u0)
nat.check(nat.load().eik_swe_krylov_bench(ctx.h, nat.dptr(u), nat.dptr(v), spec.dt, m, reps, out))
it = m * reps
N = ops.n_g
balg = N * (96 + 64 + 24) + 8 * sum(getattr(ops, k).csr.nnz for k in ("Gx","Gy","Gz","Dx","Dy","Dz","Vx","Vy","Vz","L"))
us = out[0] * 1e3 / it
print(f"{name} N={N} m={m} reps={reps}: {out[0]:.3f} ms total, {us:.1f} us/iter, keep {out[1]}, "
      f"B_alg {balg/1e6:.1f} MB -> {balg/us/1e3:.0f} GB/s ({balg/us/1e3/6543.4*100:.1f}% of 6543.4)")
nat.check(nat.load().eik_swe_info(ctx.h, info))
if info[10] and info[12] and len(sys.argv) > 4 and sys.argv[4] == "ws":
    print("WS: producer wait %.1f%% of its time, consumer wait %.1f%% of its time (+ TMA wait %.1f%%)" % (
        100 * info[9] / info[10], 100 * info[11] / info[12], 100 * info[13] / info[12]))
elif info[12]:
    tot = info[9] + info[10] + info[11]
    print("tile step cycles share: step1 %.1f%% step2 %.1f%% step3 %.1f%%, per-CTA-call avg %.0f us" % (
        100 * info[9] / tot, 100 * info[10] / tot, 100 * info[11] / tot, tot / info[12] / 1965.0))
