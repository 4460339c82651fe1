"""§8f rows 2-4 on the device: FD Jacobian check, reference solution,
convergence study with the reference's CSV schema."""

import numpy as np
import pytest

from oracle import integrate_oracle, swe_problem
from paper_1805_02144_b200.harness import (jacobian_fd_check, make_reference_solution,
                                           run_convergence_study, sphere_bundle)

pytestmark = pytest.mark.gpu


def test_fd_jacobian_check_on_device():
    b = sphere_bundle("C0")
    assert jacobian_fd_check(b.ops, b.u0, n_directions=8) <= 1e-6


def test_reference_solution_matches_oracle(tmp_path):
    b = sphere_bundle("C0")
    dts, t_end = (1800.0, 900.0), 1800.0
    ref = make_reference_solution(b, dts, t_end, cache_dir=str(tmp_path))
    again = make_reference_solution(b, dts, t_end, cache_dir=str(tmp_path))
    assert np.array_equal(ref, again)                      # cache hit
    o, _, _, _ = integrate_oracle(swe_problem(b.ops), "pexprb43", b.u0, 900.0 / 20,
                                  t_end, tol=1e-10)
    assert np.linalg.norm(ref - o) <= 1e-9 * np.linalg.norm(o)


def test_convergence_study_orders(tmp_path):
    b = sphere_bundle("C0")
    dts = (3600.0, 1800.0, 900.0, 450.0)
    rows, orders = run_convergence_study(b, ("exprb42", "epi3"), dts, 3600.0, tol=1e-10,
                                         cache_dir=str(tmp_path))
    assert len(rows) == 8
    assert orders["exprb42"] is not None and orders["exprb42"] > 3.0
    assert orders["epi3"] is not None and orders["epi3"] > 2.0
