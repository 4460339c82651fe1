"""GPU trajectories against fixtures produced by the reference itself
(tests/golden/make_golden.py) and against the oracle port run live.

Bar (BASELINE.json north_star): identical Krylov dimensions / substep counts
per engine call, relative L2 state difference <= 1e-9.
"""

import os

import numpy as np
import pytest

from oracle import integrate_oracle, swe_problem
from paper_1805_02144_b200 import swe as gswe
from paper_1805_02144_b200.states import make_config

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-9


def gold(name):
    return np.load(os.path.join(GOLD, f"{name}.npz"))


def run_gpu(ops, u0, scheme, dt, nsteps, tol):
    """Resident-state trajectory through the C ABI; per-call counters."""
    ctx = gswe.SweContext(ops)
    ctx.set_state(u0)
    ctx.reset_seeds()
    calls, steps = [], []
    for k in range(nsteps):
        sch = "rb_euler" if (scheme == "epi3" and k == 0) else scheme
        cs = ctx.step(sch, dt, tol)
        calls += [(c.substeps, c.rejections, c.matvecs, c.m_final) for c in cs]
        steps.append((sum(c.matvecs for c in cs), sum(c.substeps for c in cs)))
    return ctx.get_state(), calls, steps


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("name,scheme,steps", [
    ("c0_exprb42_24", "exprb42", 24), ("c0_pexprb43_6", "pexprb43", 6),
    ("c0_exprb53_6", "exprb53", 6), ("c0_epi3_6", "epi3", 6),
    ("c0_rb_euler_6", "rb_euler", 6)])
def test_c0_matches_reference_golden(name, scheme, steps):
    ops, u0, spec = make_config("C0")
    g = gold(name)
    assert np.array_equal(u0, g["u0"])
    u, calls, per_step = run_gpu(ops, u0, scheme, spec.dt, steps, spec.tol)
    assert [tuple(s) for s in g["steps"]] == per_step
    gc = [tuple(int(x) for x in c[1:5]) for c in g["calls"]]
    assert calls == gc
    assert rel(u, g["final"]) <= TOL


def _prefix(cfg, name, scheme, dt, steps):
    ops, u0, spec = make_config(cfg)
    g = gold(name)
    u, calls, per_step = run_gpu(ops, u0, scheme, dt, steps, 1e-8)
    assert [tuple(s) for s in g["steps"]] == per_step
    gc = [tuple(int(x) for x in c[1:5]) for c in g["calls"]]
    assert calls == gc
    idx = g["sample_idx"]
    assert np.max(np.abs(u[idx] - g["final_sample"])) <= TOL * np.max(np.abs(g["final_sample"]))
    assert abs(np.linalg.norm(u) - float(g["final_norm"])) <= TOL * float(g["final_norm"])
    fn = np.array([np.linalg.norm(a) for a in np.split(u, 4)])
    assert np.all(np.abs(fn - g["final_field_norms"]) <= 1e-8 * g["final_field_norms"] + 1e-12)
    return ops, u0, u


def test_c1_pexprb43_prefix_matches_reference_golden():
    ops, u0, u = _prefix("C1", "c1_pexprb43_2", "pexprb43", 1800.0, 2)
    # full state against the oracle port, live (L6: a few seconds of CPU)
    ref, _, _, _ = integrate_oracle(swe_problem(ops), "pexprb43", u0, 1800.0, 3600.0,
                                    tol=1e-8)
    assert rel(u, ref) <= TOL


@pytest.mark.slow
def test_c2_exprb53_prefix_matches_reference_golden():
    _prefix("C2", "c2_exprb53_1", "exprb53", 1800.0, 1)


@pytest.mark.slow
def test_c3_exprb42_prefix_matches_reference_golden():
    _prefix("C3", "c3_exprb42_1", "exprb42", 600.0, 1)


@pytest.mark.slow
def test_c3_epi3_prefix_matches_reference_golden():
    _prefix("C3", "c3_epi3_2", "epi3", 600.0, 2)


def test_c0_long_run_matches_oracle_live():
    """The whole C0 run (24 exprb42 steps) through integrate() (Python shim,
    state copied every step) equals the oracle port's."""
    from paper_1805_02144_b200.integrators import integrate, swe_problem as gprob
    ops, u0, spec = make_config("C0")
    recs = integrate(gprob(ops), "exprb42", u0, spec.dt, spec.steps * spec.dt, tol=spec.tol)
    ref, steps, _, _ = integrate_oracle(swe_problem(ops), "exprb42", u0, spec.dt,
                                        spec.steps * spec.dt, tol=spec.tol)
    assert [(r.matvecs, r.substeps) for r in recs[1:]] == steps
    assert rel(recs[-1].u, ref) <= TOL


@pytest.mark.slow
@pytest.mark.parametrize("dt", [900.0, 3600.0, 7200.0])
def test_c1_dt_sweep_matches_oracle(dt):
    """C1's dt sweep (pEXPRB4): two steps per dt, full state and per-call
    counters against the oracle port run live (L6)."""
    ops, u0, _ = make_config("C1")
    u, calls, per_step = run_gpu(ops, u0, "pexprb43", dt, 2, 1e-8)
    ref, steps, _, log = integrate_oracle(swe_problem(ops), "pexprb43", u0, dt, 2 * dt,
                                          tol=1e-8)
    assert per_step == steps
    assert calls == [(c[1], c[2], c[3], c[4]) for c in log.calls]
    assert rel(u, ref) <= TOL


@pytest.mark.slow
def test_c4_l9_exprb42_first_step_matches_reference_golden():
    """C4 at L9 (2.6M cells): the cold-start EXPRB4 step (rejections and the
    m jump) against the reference run on the CPU (207 s there)."""
    _prefix("C4", "c4_exprb42_1", "exprb42", 900.0, 1)
