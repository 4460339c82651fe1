"""Every BASELINE.json configuration run at its full length on the device
(resident state, CUDA-graph steps): device time, steps/s, Krylov iterations,
mass / energy drift (area-weighted diagnostics of the initial and final states).

    python tools/run_configs.py [out.txt]
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1805_02144_b200 import swe as gswe  # noqa: E402
from paper_1805_02144_b200.states import CONFIGS, make_config  # noqa: E402

RUNS = [  # (config, level, scheme, dt, steps) -- BASELINE.json configs 0-4
    ("C0", None, "exprb42", 3600.0, 24),
    ("C1", None, "pexprb43", 900.0, 96),
    ("C1", None, "pexprb43", 1800.0, 48),
    ("C1", None, "pexprb43", 3600.0, 24),
    ("C1", None, "pexprb43", 7200.0, 12),
    ("C2", None, "exprb53", 1800.0, 240),
    ("C3", None, "exprb42", 600.0, 144),
    ("C3", None, "epi3", 600.0, 144),
    ("C4", 9, "exprb42", 900.0, 10),
    ("C4", 9, "exprb53", 900.0, 10),
]


def run(cfg, level, scheme, dt, nsteps):
    ops, u0, spec = make_config(cfg, level=level)
    ctx = gswe.SweContext(ops)
    ctx.set_state(u0)
    ctx.reset_seeds()
    d0 = gswe.diagnostics(ops, state=u0, area_weighted=True)
    ms, iters = 0.0, 0
    k0 = ctx.krylov_iters()
    t0 = time.perf_counter()
    for k in range(nsteps):
        sch = "rb_euler" if (scheme == "epi3" and k == 0) else scheme
        ctx.step(sch, dt, spec.tol)
        ms += ctx.last_kernel_ms()
    wall = time.perf_counter() - t0
    iters = ctx.krylov_iters() - k0
    u = ctx.get_state()
    d1 = gswe.diagnostics(ops, state=u, area_weighted=True)
    return (f"{cfg} L{ops.level} ({ops.n_g} cells) {scheme} dt={dt:g}s x{nsteps} "
            f"(t_end {nsteps * dt / 86400:.2f} d): device {ms:.1f} ms = {1e3 * nsteps / ms:.1f} "
            f"steps/s (wall {wall:.2f} s), {iters / nsteps:.1f} Krylov iters/step, "
            f"mass drift {(d1.mass - d0.mass) / d0.mass:+.2e}, energy drift "
            f"{(d1.energy - d0.energy) / d0.energy:+.2e}, finite {bool(np.isfinite(u).all())}")


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    lines = [run(*r) for r in RUNS]
    txt = "\n".join(lines)
    print(txt)
    if out:
        with open(out, "w") as fh:
            fh.write("tools/run_configs.py: every BASELINE.json config at full length on one B200 "
                     "(resident state, graph-replayed steps, device time from CUDA events)\n"
                     + txt + "\n")


if __name__ == "__main__":
    main()
