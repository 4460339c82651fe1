"""Round 1's bench window on the current build: C3 EXPRB4, trajectory steps
6-25 from the seeded initial state (5 untimed steps, then 20 timed ones,
warm engine seeds), device time of the step graphs.

    python tools/warm_window.py
"""
import sys

sys.path.insert(0, ".")
from paper_1805_02144_b200 import swe as gswe  # noqa: E402
from paper_1805_02144_b200.states import make_config  # noqa: E402

ops, u0, spec = make_config("C3")
ctx = gswe.SweContext(ops)
ctx.set_state(u0)
for _ in range(5):
    ctx.step("exprb42", spec.dt, spec.tol)
k0 = ctx.krylov_iters()
ms = 0.0
mv = 0
for _ in range(20):
    calls = ctx.step("exprb42", spec.dt, spec.tol)
    ms += ctx.last_kernel_ms()
    mv += sum(int(c.matvecs) for c in calls)
it = ctx.krylov_iters() - k0
print(f"C3 exprb42 steps 6-25: {ms / 20:.3f} ms/step = {20e3 / ms:.1f} steps/s, "
      f"{it / 20:.1f} Krylov iterations/step, {mv / 20:.1f} matvecs/step "
      f"(round 1, r01l: 8.03-8.13 ms/step = 123.1-124.5 steps/s, 64.8 iterations/step)")
