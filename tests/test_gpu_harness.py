"""§8f rows 2-4 on the device: the study harness and CLI (reference
pkg/tests/test_harness.py restated), the FD Jacobian check, reference
solutions, and a sphere-config CLI run whose counters equal the reference's
own golden run."""

import os

import numpy as np
import pytest

from oracle import integrate_oracle, swe_problem
from paper_1805_02144_b200 import cli
from paper_1805_02144_b200.harness import (CSV_HEADER, StudyConfig, jacobian_fd_check,
                                           make_problem, make_reference_solution,
                                           run_convergence_study, sphere_bundle)

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_fd_jacobian_check_on_device():
    b = sphere_bundle("C0")
    cfg = StudyConfig(problem="sphere_C0")
    assert jacobian_fd_check(cfg, n_directions=8, state=b.u0, ops=b.ops) <= 1e-6
    # planar default (the reference's check-jacobian problem) and its mutation
    assert jacobian_fd_check(StudyConfig(problem="swe_planar"), n_directions=6) <= 1e-5
    assert jacobian_fd_check(StudyConfig(problem="swe_planar"), n_directions=6,
                             corrupt=True) > 1e-3


def test_reference_solution_matches_oracle(tmp_path):
    cfg = StudyConfig(problem="sphere_C0", schemes=("exprb42",), dts=(1800.0, 900.0),
                      t_end=1800.0, cache_dir=str(tmp_path))
    b = make_problem(cfg)
    ref = make_reference_solution(cfg, b)
    assert len(list(tmp_path.glob("ref_*.npy"))) == 1
    assert np.array_equal(ref, make_reference_solution(cfg, b))  # cache hit
    o, _, _, _ = integrate_oracle(swe_problem(b.ops), "pexprb43", b.u0, 900.0 / 20, 1800.0,
                                  tol=1e-10)
    assert np.linalg.norm(ref - o) <= 1e-9 * np.linalg.norm(o)


def test_reference_solution_cached_rd(tmp_path):
    """test_harness.py:112-121 (reaction-diffusion: host F/J, device engine)."""
    cfg = StudyConfig(problem="reaction_diffusion_1d", schemes=("rb_euler",),
                      dts=(0.5, 0.25, 0.125, 0.0625), t_end=0.25, tol=1e-6,
                      cache_dir=str(tmp_path))
    bundle = make_problem(cfg)
    ref1 = make_reference_solution(cfg, bundle)
    assert len(list(tmp_path.glob("ref_*.npy"))) == 1
    assert np.array_equal(ref1, make_reference_solution(cfg, bundle))


def test_reference_uses_exact_when_available():
    cfg = StudyConfig(problem="manufactured", schemes=("rb_euler",),
                      dts=(0.1, 0.05, 0.025, 0.0125), t_end=1.0)
    bundle = make_problem(cfg)
    assert np.array_equal(make_reference_solution(cfg, bundle), bundle.problem.exact(1.0))


def test_convergence_study_requires_enough_dts():
    cfg = StudyConfig(problem="manufactured", schemes=("rb_euler",), dts=(0.1, 0.05),
                      t_end=1.0)
    with pytest.raises(ValueError):
        run_convergence_study(cfg)


def test_convergence_study_orders_on_sphere(tmp_path):
    cfg = StudyConfig(problem="sphere_C0", schemes=("exprb42", "epi3"),
                      dts=(3600.0, 1800.0, 900.0, 450.0), t_end=3600.0, tol=1e-10,
                      cache_dir=str(tmp_path))
    rows, orders = run_convergence_study(cfg)
    assert len(rows) == 8
    assert orders["exprb42"] is not None and orders["exprb42"] > 3.0
    assert orders["epi3"] is not None and orders["epi3"] > 2.0


def test_cli_converge_writes_csv(tmp_path):
    out = tmp_path / "rows.csv"
    status = cli.main(["converge", "--problem", "manufactured", "--schemes", "rb_euler",
                       "--dts", "0.2,0.1,0.05,0.025", "--t-end", "0.4", "--tol", "1e-8",
                       "--out", str(out)])
    assert status == 0
    lines = out.read_text().strip().splitlines()
    assert lines[0] == CSV_HEADER and len(lines) == 5


def test_cli_run_single(capsys):
    status = cli.main(["run", "--problem", "manufactured", "--schemes", "rb_euler",
                       "--dts", "0.1", "--t-end", "0.2", "--tol", "1e-8"])
    assert status == 0
    assert capsys.readouterr().out.startswith(CSV_HEADER)


def test_cli_run_rejects_multiple_schemes():
    assert cli.main(["run", "--problem", "manufactured", "--schemes", "rb_euler,epi3",
                     "--dts", "0.1", "--t-end", "0.2"]) == 2


def test_cli_check_jacobian():
    assert cli.main(["check-jacobian"]) == 0


def test_cli_run_sphere_c0_matches_reference_counters(tmp_path):
    """The CLI on BASELINE config C0 (EXPRB4, 24 x 3600 s, tol 1e-8): the CSV
    row's steps / matvecs / substeps equal the reference's own run
    (tests/golden/c0_exprb42_24.npz, made by the unmodified reference)."""
    out = tmp_path / "c0.csv"
    status = cli.main(["run", "--problem", "sphere_C0", "--schemes", "exprb42",
                       "--dts", "3600", "--t-end", "86400", "--tol", "1e-8",
                       "--out", str(out)])
    assert status == 0
    header, row = out.read_text().strip().splitlines()
    assert header == CSV_HEADER
    f = row.split(",")
    g = np.load(os.path.join(GOLD, "c0_exprb42_24.npz"))
    assert f[0] == "exprb42" and f[1] == "3600"
    assert (int(f[4]), int(f[5]), int(f[6])) == (24, int(g["steps"][:, 0].sum()),
                                                 int(g["steps"][:, 1].sum()))
    assert 0.0 < float(f[2]) < 1e-3
