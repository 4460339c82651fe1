"""Long-run golden fixtures: the REFERENCE (/root/reference) run for the full
length each BASELINE.json config states, on our sphere operators and seeded
states (test infrastructure; nothing here ships).

    python tests/golden/make_long_golden.py C3:exprb42:600:144 [CFG:SCHEME:DT:STEPS[:LEVEL] ...]

Each job writes tests/golden/long_<cfg>[l<level>]_<scheme>_<dt>.npz holding
  * every engine call of the run: step index, p, substeps, rejections,
    matvecs, m_final, tau_final (the decision trace the GPU must reproduce);
  * per-step (matvecs, substeps) and per-step field norms;
  * at checkpoint steps {1, 2, 4, ..., final}: CountSketches of the state
    (tests/golden/sketch.py) and sampled entries (4096 at the final step,
    1024 before), so the device trajectory is compared against the whole
    reference state along the run.
Runs with OPENBLAS_NUM_THREADS=1 so several jobs share the host.
"""

import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from expintkit import integrators as R  # noqa: E402
from expintkit import swe as RS  # noqa: E402

from make_golden import ops_digest  # noqa: E402
from paper_1805_02144_b200.states import make_config  # noqa: E402
from sketch import field_norms, sample_idx, sketch  # noqa: E402


def checkpoints(nsteps):
    c, k = [], 1
    while k < nsteps:
        c.append(k)
        k *= 2
    return c + [nsteps]


def fixture_name(cfg, scheme, dt, level=None):
    lv = "" if level is None else f"l{level}"
    return f"long_{cfg.lower()}{lv}_{scheme}_{int(dt)}"


def run(cfg, scheme, dt, nsteps, tol=1e-8, level=None):
    ops, u0, spec = make_config(cfg, level)
    n = 4 * ops.n_g
    cps = checkpoints(nsteps)
    idx_f = sample_idx(n, 4096)
    idx_c = idx_f[:1024]
    state = {"step": 0}
    calls = []
    orig = R.phipm_simul_iom2

    def spy(task):
        res = orig(task)
        calls.append((state["step"] + 1, len(task.v) - 1, res.substeps, res.rejections,
                      res.matvecs, res.m_final, res.tau_final))
        return res

    per_step, norms, sk, samp = [], [], [], []
    t0 = time.time()

    def obs(rec):
        if rec.dt == 0.0:
            return
        state["step"] += 1
        k = state["step"]
        per_step.append((rec.matvecs, rec.substeps))
        norms.append(field_norms(rec.u))
        if k in cps:
            sk.append(sketch(rec.u))
            samp.append(rec.u[idx_f if k == nsteps else idx_c])
            print(f"  {cfg} {scheme} dt={dt:g}: step {k}/{nsteps} "
                  f"{time.time() - t0:.0f}s", flush=True)

    R.phipm_simul_iom2 = spy
    prob = R.SemilinearProblem(n=n, f=lambda u: RS.rhs(ops, u),
                               jac=lambda u: RS.assemble_jacobian(ops, u))
    try:
        recs = R.integrate(prob, scheme, u0, dt, nsteps * dt, tol=tol, observers=(obs,))
    finally:
        R.phipm_simul_iom2 = orig
    secs = time.time() - t0
    u = recs[-1].u
    del recs
    name = fixture_name(cfg, scheme, dt, level)
    out = dict(
        digest=np.array(ops_digest(ops)), cfg=np.array(cfg), scheme=np.array(scheme),
        dt=dt, nsteps=nsteps, tol=tol, cpu_seconds=secs,
        calls=np.array(calls, dtype=float), steps=np.array(per_step, dtype=np.int64),
        field_norms=np.array(norms), checkpoints=np.array(cps),
        sketches=np.array(sk), final_norm=np.linalg.norm(u),
        sample_idx=idx_f, final_sample=samp[-1],
        cp_samples=np.array(samp[:-1]) if len(samp) > 1 else np.zeros((0, 1024)))
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {nsteps} steps, {len(calls)} calls, {secs:.0f}s, "
          f"{os.path.getsize(path)} bytes", flush=True)


def main():
    for job in sys.argv[1:]:
        parts = job.split(":")
        cfg, scheme, dt, nsteps = parts[0], parts[1], float(parts[2]), int(parts[3])
        level = int(parts[4]) if len(parts) > 4 else None
        run(cfg, scheme, dt, nsteps, level=level)


if __name__ == "__main__":
    main()
