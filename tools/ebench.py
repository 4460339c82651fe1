"""Engine-call benchmark: one phipm call (A = dt J(u0)) at a config, device
time per Krylov iteration vs the bare Krylov-loop microbenchmark."""
import sys, ctypes as C
import numpy as np
sys.path.insert(0, ".")
from paper_1805_02144_b200.states import make_config
from paper_1805_02144_b200 import swe as gswe, _native as nat
from paper_1805_02144_b200.phipm import PhiTask, phipm_simul_iom2
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
ops, u0, spec = make_config(name)
ctx = gswe.context(ops)
f = ctx.rhs(u0)
A = gswe.assemble_jacobian(ops, u0).scaled(spec.dt)
v = [np.zeros_like(u0), spec.dt * f]
buf = (C.c_double * 16)()
lib = nat.load()
for m0 in (40, 40, 60):
    lib.eik_prof_read(buf, 1)
    it0 = ctx.krylov_iters()
    res = phipm_simul_iom2(PhiTask(A=A, v=v, rho=[0.75], tol=1e-8, m_init=m0, tau_init=0.75))
    it = ctx.krylov_iters() - it0
    ms = ctx.last_kernel_ms()
    print(f"m_init {m0}: {ms:.3f} ms, krylov {it}, matvecs {res.matvecs}, substeps {res.substeps}, "
          f"rej {res.rejections} -> {ms*1e3/it:.1f} us per Krylov iteration (whole call)")
    if lib.eik_prof_read(buf, 1) == 0:
        tot = sum(buf[k] for k in range(8))
        print(f"   krylov phase {buf[3] / tot * ms * 1e3 / it:.1f} us/iter, dense {buf[4] / tot * ms * 1e3:.0f} us, "
              f"cand {buf[5] / tot * ms * 1e3:.0f} us, wrec {buf[2] / tot * ms * 1e3:.0f} us")
