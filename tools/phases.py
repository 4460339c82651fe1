"""Per-phase clock shares of the step kernel (build with -DEIK_PROF=1) at a
config: python tools/phases.py [C3] [steps]."""
import sys, ctypes as C
import numpy as np
sys.path.insert(0, ".")
from paper_1805_02144_b200.states import make_config
from paper_1805_02144_b200 import swe as gswe, _native as nat
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
ops, u0, spec = make_config(name)
ctx = gswe.SweContext(ops)
lib = nat.load()
ctx.set_state(u0)
for _ in range(2):
    ctx.step(spec.scheme, spec.dt, spec.tol)
buf = (C.c_double * 16)()
lib.eik_prof_read(buf, 1)
k0 = ctx.krylov_iters()
e0 = lib.eik_swe_explicit_orth(ctx.h)
ms = 0.0
for _ in range(steps):
    ctx.step(spec.scheme, spec.dt, spec.tol)
    ms += ctx.last_kernel_ms()
prof = lib.eik_prof_read(buf, 1) == 0
it = ctx.krylov_iters() - k0
eo = lib.eik_swe_explicit_orth(ctx.h) - e0
names = ["rhs", "nnz", "wrec", "krylov", "dense", "cand", "dev", "misc"]
tot = sum(buf[k] for k in range(8))
print(f"{name}: {ms/steps:.3f} ms/step, {it/steps:.1f} Krylov iters/step, "
      f"{ms*1e3/it:.1f} us per iter incl. everything, explicit-orth passes/step {eo/steps:.1f}")
if not prof or tot == 0:
    sys.exit(0)
print("  " + "  ".join(f"{n} {100*buf[k]/tot:.1f}%" for k, n in enumerate(names)))
kr = buf[3] / tot * ms * 1e3 / it
print(f"  krylov phase: {kr:.1f} us per iteration")
