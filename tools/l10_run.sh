# C4 at L10 (10,485,762 cells): grid build + 2 EXPRB4 steps + 1 EXPRB5 step
mkdir -p gpurun_out
python - > gpurun_out/l10.log 2>&1 <<'PY'
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_1805_02144_b200.states import make_config
from paper_1805_02144_b200 import swe as gswe
t = time.time()
ops, u0, spec = make_config("C4", level=10)
print(f"grid L10 N={ops.n_g} built in {time.time()-t:.0f}s", flush=True)
t = time.time()
ctx = gswe.SweContext(ops)
print(f"context created in {time.time()-t:.0f}s", flush=True)
ctx.set_state(u0)
for k, sch in enumerate(["exprb42", "exprb42", "exprb53"]):
    it0 = ctx.krylov_iters()
    calls = ctx.step(sch, 900.0, 1e-8)
    it = ctx.krylov_iters() - it0
    ms = ctx.last_kernel_ms()
    print(f"{sch} step {k}: {ms:.1f} ms, krylov {it}, {ms*1e3/max(it,1):.0f} us/iter, "
          f"calls {[(c.substeps, c.rejections, c.matvecs, c.m_final) for c in calls]}", flush=True)
u = ctx.get_state()
print("finite", bool(np.isfinite(u).all()))
PY
echo rc=$?
