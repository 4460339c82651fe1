"""Quick GPU probe: per-step device time and Krylov iterations for a config."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1805_02144_b200.states import make_config
from paper_1805_02144_b200 import swe as gswe

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
scheme = sys.argv[2] if len(sys.argv) > 2 else "exprb42"
nsteps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
t0 = time.time()
ops, u0, spec = make_config(name)
print(f"grid L{ops.level} N={ops.n_g} built in {time.time()-t0:.1f}s", flush=True)
ctx = gswe.context(ops)
ctx.set_state(u0)
for k in range(nsteps):
    it0 = ctx.krylov_iters()
    t = time.time()
    calls = ctx.step(scheme if not (scheme == "epi3" and k == 0) else "rb_euler", spec.dt, spec.tol)
    wall = time.time() - t
    it = ctx.krylov_iters() - it0
    ms = ctx.last_kernel_ms()
    mv = sum(c.matvecs for c in calls)
    print(f"step {k}: {ms:8.3f} ms device, wall {wall*1e3:8.2f} ms, matvecs {mv}, krylov {it}, "
          f"{ms/max(it,1)*1e3:7.1f} us/iter, calls {[ (c.substeps, c.rejections, c.matvecs, c.m_final) for c in calls]}", flush=True)
import ctypes
from paper_1805_02144_b200 import _native as nat
print("explicit orthogonalisation passes:", nat.load().eik_swe_explicit_orth(ctx.h), "of", ctx.krylov_iters())
pr = (ctypes.c_double * 16)()
if nat.load().eik_prof_read(pr, 1) == 0:
    names = ["rhs", "nnz", "wrec", "krylov", "dense", "cand", "dev", "misc"]
    tot = sum(pr[:8])
    print("phase share (CTA0 cycles, all steps):", ", ".join(f"{n} {100*pr[k]/tot:.1f}%" for k, n in enumerate(names)),
          f"total {tot/1.965e6:.1f} ms")
u = ctx.get_state()
print("finite", np.isfinite(u).all(), "h range", u[3*ops.n_g:].min(), u[3*ops.n_g:].max())
