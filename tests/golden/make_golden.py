"""Generate golden fixtures by running the REFERENCE (/root/reference) itself.

The reference package has no sphere grid and pins nothing at sphere scale
(SURVEY.md §8c), so parity on BASELINE.json's configs is pinned here: the
unmodified reference ``integrate`` / ``phipm_simul_iom2`` run on our sphere
``DiscreteOperators`` and seeded states, and the results are stored as small
.npz fixtures that travel to the GPU box (where /root/reference does not).

    python tests/golden/make_golden.py [--big] [--c4]

Writes tests/golden/*.npz.  ``--big`` adds the L7/L8 prefixes (minutes),
``--c4`` the L9 first step.  The full-length runs of every config are made
by make_long_golden.py.
"""

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from expintkit import integrators as R  # noqa: E402
from expintkit import swe as RS  # noqa: E402

from paper_1805_02144_b200.states import make_config  # noqa: E402

SAMPLE = 64


def ops_digest(ops):
    h = hashlib.sha256()
    for name in ("Gx", "Gy", "Gz", "Dx", "Dy", "Dz", "Vx", "Vy", "Vz", "L", "Df"):
        c = getattr(ops, name).csr
        h.update(np.ascontiguousarray(c.indptr).tobytes())
        h.update(np.ascontiguousarray(c.indices).tobytes())
        h.update(np.ascontiguousarray(c.data).tobytes())
    for f in ("n_x", "n_y", "n_z", "f", "h_s"):
        h.update(np.ascontiguousarray(getattr(ops, f)).tobytes())
    return h.hexdigest()


def run_reference(ops, u0, scheme, dt, nsteps, tol):
    """Reference integrate() with every engine call recorded."""
    calls = []
    orig = R.phipm_simul_iom2

    def spy(task):
        res = orig(task)
        calls.append((len(task.v) - 1, res.substeps, res.rejections,
                      res.matvecs, res.m_final, res.tau_final))
        return res

    R.phipm_simul_iom2 = spy
    try:
        prob = R.SemilinearProblem(n=4 * ops.n_g, f=lambda u: RS.rhs(ops, u),
                                   jac=lambda u: RS.assemble_jacobian(ops, u))
        t = time.time()
        recs = R.integrate(prob, scheme, u0, dt, nsteps * dt, tol=tol)
        secs = time.time() - t
    finally:
        R.phipm_simul_iom2 = orig
    return recs, np.array(calls, dtype=float), secs


def save(name, ops, u0, recs, calls, secs, full_state):
    u = recs[-1].u
    rng = np.random.default_rng(12345)
    idx = np.sort(rng.choice(u.shape[0], size=min(SAMPLE, u.shape[0]), replace=False))
    out = dict(
        digest=np.array(ops_digest(ops)),
        u0_norm=np.linalg.norm(u0), u0_sample=u0[idx],
        steps=np.array([(r.matvecs, r.substeps) for r in recs[1:]]),
        calls=calls, final_norm=np.linalg.norm(u), sample_idx=idx,
        final_sample=u[idx], cpu_seconds=secs,
        final_field_norms=np.array([np.linalg.norm(a) for a in np.split(u, 4)]))
    if full_state:
        out["u0"] = u0
        out["final"] = u
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {len(recs) - 1} steps, {secs:.1f}s, {os.path.getsize(path)} bytes",
          flush=True)


def main():
    big = "--big" in sys.argv
    ops, u0, spec = make_config("C0")
    recs, calls, secs = run_reference(ops, u0, "exprb42", spec.dt, spec.steps, spec.tol)
    save("c0_exprb42_24", ops, u0, recs, calls, secs, True)
    for scheme in ("pexprb43", "exprb53", "epi3", "rb_euler"):
        recs, calls, secs = run_reference(ops, u0, scheme, spec.dt, 6, spec.tol)
        save(f"c0_{scheme}_6", ops, u0, recs, calls, secs, True)
    ops, u0, spec = make_config("C1")
    recs, calls, secs = run_reference(ops, u0, "pexprb43", 1800.0, 2, 1e-8)
    save("c1_pexprb43_2", ops, u0, recs, calls, secs, False)
    if big:
        ops, u0, spec = make_config("C2")
        recs, calls, secs = run_reference(ops, u0, "exprb53", 1800.0, 1, 1e-8)
        save("c2_exprb53_1", ops, u0, recs, calls, secs, False)
        ops, u0, spec = make_config("C3")
        recs, calls, secs = run_reference(ops, u0, "exprb42", 600.0, 1, 1e-8)
        save("c3_exprb42_1", ops, u0, recs, calls, secs, False)
        recs, calls, secs = run_reference(ops, u0, "epi3", 600.0, 2, 1e-8)
        save("c3_epi3_2", ops, u0, recs, calls, secs, False)
    if "--c4" in sys.argv:
        # C4 at L9 (2.6 M cells): the cold-start EXPRB4 step (~210 s here)
        ops, u0, spec = make_config("C4")
        recs, calls, secs = run_reference(ops, u0, "exprb42", 900.0, 1, 1e-8)
        save("c4_exprb42_1", ops, u0, recs, calls, secs, False)


if __name__ == "__main__":
    main()
