"""Study-driver logic that needs no device, restating the reference's
pkg/tests/test_harness.py (the parts that do not integrate), plus the CSV
format pinned against the reference's own ResultRow."""

import numpy as np
import pytest

from paper_1805_02144_b200.harness import (CSV_HEADER, ResultRow, StudyConfig, fit_order,
                                           make_manufactured, parse_config,
                                           rel_linf_error, write_csv)


def test_parse_config(tmp_path):
    path = tmp_path / "cfg.txt"
    path.write_text("# comment\nnx = 16\n\nh0=7000.5\nname = hill run\n")
    assert parse_config(path) == {"nx": "16", "h0": "7000.5", "name": "hill run"}
    bad = tmp_path / "bad.txt"
    bad.write_text("no equals sign here\n")
    with pytest.raises(ValueError):
        parse_config(bad)


def test_study_config_validation():
    with pytest.raises(ValueError):
        StudyConfig(problem="nope")
    with pytest.raises(ValueError):
        StudyConfig(schemes=("rb_euler", "bogus"))
    with pytest.raises(ValueError):
        StudyConfig(dts=(0.1, 0.2))
    assert StudyConfig(problem="sphere_C3", dts=(600,)).dts == (600.0,)


def test_csv_schema(tmp_path):
    rows = [ResultRow("rb_euler", 0.1, 1e-4, 0.1, 10, 50, 12)]
    p = tmp_path / "out.csv"
    write_csv(rows, p)
    lines = p.read_text().strip().splitlines()
    assert lines[0] == CSV_HEADER == "scheme,dt,error_linf,cpu_seconds,steps,matvecs,substeps"
    assert lines[1].startswith("rb_euler,0.1,")


@pytest.mark.reference
def test_csv_rows_byte_equal_to_reference_writer(reference, tmp_path):
    """The same rows written by the reference's write_csv and by ours are
    byte-identical (harness.py:84-97, 356-360)."""
    from expintkit import harness as RH
    vals = [("exprb42", 3600.0, 1.234567890123e-7, 0.0123456, 24, 1520, 48),
            ("epi3", 0.025, 1e-14, 12.5, 40, 999, 40),
            ("pexprb43", 1.0 / 3.0, 3.3e-3, 1.0, 3, 7, 3)]
    a, b = tmp_path / "ours.csv", tmp_path / "ref.csv"
    write_csv([ResultRow(*v) for v in vals], a)
    RH.write_csv([RH.ResultRow(*v) for v in vals], b)
    assert a.read_bytes() == b.read_bytes()
    assert CSV_HEADER == RH.CSV_HEADER


def test_fit_order_slopes():
    dts = [0.1, 0.05, 0.025, 0.0125]
    rows = [ResultRow("s", d, 0.5 * d ** 3, 0, 1, 1, 1) for d in dts]
    slope, flagged = fit_order(rows, 1e-12)
    assert slope == pytest.approx(3.0, abs=1e-10) and not flagged
    rows = [ResultRow("s", d, d ** 2, 0, 1, 1, 1) for d in dts[:3]]
    rows.append(ResultRow("s", dts[3], 1e-14, 0, 1, 1, 1))
    slope, flagged = fit_order(rows, 1e-12)
    assert slope == pytest.approx(2.0, abs=1e-10) and len(flagged) == 1
    assert fit_order(rows[:2], 1e-12)[0] is None


def test_rel_linf_error_with_slice():
    u = np.array([1.0, 2.0, 5.0, 8.0])
    ref = np.array([1.0, 2.0, 4.0, 8.0])
    assert rel_linf_error(u, ref) == pytest.approx(1.0 / 8.0)
    assert rel_linf_error(u, ref, slice(2, 4)) == pytest.approx(1.0 / 8.0)
    assert rel_linf_error(u, ref, slice(0, 2)) == 0.0


def test_manufactured_exact_solution_satisfies_ode():
    problem = make_manufactured(seed=0).problem
    for t in (0.0, 0.3, 0.8):
        u = problem.exact(t)
        h = 1e-6
        dudt = (problem.exact(t + h) - problem.exact(t - h)) / (2 * h)
        assert np.max(np.abs(dudt - problem.rhs(u))) <= 1e-6 * max(1.0, np.max(np.abs(dudt)))


def test_manufactured_jacobian_matches_fd():
    problem = make_manufactured(seed=0).problem
    u = problem.exact(0.4)
    J = problem.jacobian(u).toarray()
    rng = np.random.default_rng(3)
    for _ in range(5):
        d = rng.standard_normal(problem.n)
        d /= np.linalg.norm(d)
        fd = (problem.rhs(u + 1e-7 * d) - problem.rhs(u - 1e-7 * d)) / 2e-7
        assert np.max(np.abs(J @ d - fd)) <= 1e-5 * max(1.0, np.max(np.abs(fd)))


@pytest.mark.reference
def test_problems_equal_reference_problems(reference):
    """The restated study problems build the reference's operators/states."""
    from expintkit import harness as RH
    from expintkit import swe as RS
    from paper_1805_02144_b200 import harness as H
    from paper_1805_02144_b200 import swe as S
    a, b = H.make_manufactured(0), RH.make_manufactured(0)
    assert np.array_equal(a.u0, b.u0)
    z = a.u0 + 0.1
    assert np.array_equal(a.problem.f(z), b.problem.f(z))
    assert np.array_equal(a.problem.jac(z).toarray(), b.problem.jac(z).toarray())
    a, b = H.make_reaction_diffusion(0), RH.make_reaction_diffusion(0)
    assert np.array_equal(a.u0, b.u0)
    assert np.array_equal(a.problem.f(a.u0), b.problem.f(b.u0))
    ops_a = S.planar_periodic_operators(16, 12, 1e5)
    ops_b = RS.planar_periodic_operators(16, 12, 1e5)
    for name in ("Gx", "Gy", "Gz", "Dx", "Dy", "Dz", "Vx", "Vy", "Vz", "L", "Df"):
        ca, cb = getattr(ops_a, name).csr, getattr(ops_b, name).csr
        assert (ca != cb).nnz == 0 and ca.nnz == cb.nnz
    assert ops_a.nu == ops_b.nu
    assert np.array_equal(S.gaussian_hill_state(ops_a, 16, 12, 1e5),
                          RS.gaussian_hill_state(ops_b, 16, 12, 1e5))
