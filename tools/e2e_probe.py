import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1805_02144_b200.states import make_config
from paper_1805_02144_b200 import swe as gswe, _native as nat
ops, u0, spec = make_config("C3")
ctx = gswe.SweContext(ops)
ctx.set_state(u0)
for _ in range(3): ctx.step("exprb42", spec.dt, spec.tol)
pins = [torch.empty(4 * ops.n_g, dtype=torch.float64).pin_memory() for _ in range(2)]
bufs = [p.numpy() for p in pins]
bufs[0][:] = ctx.get_state()
T = {"set": 0.0, "step": 0.0, "get": 0.0}
for k in range(6):
    hin, hout = bufs[k & 1], bufs[(k + 1) & 1]
    t0 = time.perf_counter(); ctx.set_state(hin); t1 = time.perf_counter()
    ctx.step("exprb42", spec.dt, spec.tol); t2 = time.perf_counter()
    nat.check(nat.load().eik_swe_get_state(ctx.h, nat.dptr(hout)), "get"); t3 = time.perf_counter()
    if k >= 1:
        T["set"] += t1 - t0; T["step"] += t2 - t1; T["get"] += t3 - t2
    print(f"set {1e3*(t1-t0):.2f} ms step {1e3*(t2-t1):.2f} ms (kernel {ctx.last_kernel_ms():.2f}) get {1e3*(t3-t2):.2f} ms")
