"""GPU parity against the CPU oracle (oracle/) on identical seeded inputs."""

import numpy as np
import pytest

from oracle import (OracleOperator, engine_run, integrate_oracle, swe_jacobian,
                    swe_jv_matrix_free, swe_problem, swe_rhs)
from paper_1805_02144_b200 import swe as gswe
from paper_1805_02144_b200.integrators import integrate, swe_problem as gpu_problem
from paper_1805_02144_b200.phipm import PhiTask, phipm_simul_iom2
from paper_1805_02144_b200.states import make_config

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def c0():
    return make_config("C0")


def test_rhs_matches_oracle(c0):
    ops, u0, _ = c0
    assert rel(gswe.rhs(ops, u0), swe_rhs(ops, u0)) <= 1e-12


def test_jv_matches_assembled_oracle(c0):
    ops, u0, _ = c0
    rng = np.random.default_rng(5)
    J = swe_jacobian(ops, u0)
    for _ in range(3):
        v = rng.standard_normal(4 * ops.n_g)
        got = gswe.assemble_jacobian(ops, u0).matvec(v)
        assert rel(got, J.matvec(v)) <= 1e-13


def test_nnz_matches_scipy(c0):
    ops, u0, _ = c0
    J = swe_jacobian(ops, u0).csr
    N = ops.n_g
    ref_rows = np.diff(J.indptr).reshape(4, N).sum(0)
    import ctypes
    from paper_1805_02144_b200 import _native as nat
    ctx = gswe.context(ops)
    per = np.zeros(N)
    tot = ctypes.c_int64(0)
    u = np.ascontiguousarray(u0)
    nat.check(nat.load().eik_swe_jac_nnz_rows(ctx.h, nat.dptr(u), ctypes.byref(tot), nat.dptr(per)))
    bad = np.flatnonzero(per != ref_rows)
    print("bad cells", bad[:20], per[bad[:20]], ref_rows[bad[:20]], "deg", ops.mesh.deg[bad[:20]])
    assert tot.value == J.nnz


def test_csr_engine_matches_oracle():
    rng = np.random.default_rng(23)
    n = 40
    Q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    A = Q @ np.diag(-np.logspace(0, 3, n)) @ Q.T
    v = [rng.standard_normal(n) for _ in range(4)]
    rho = [0.25, 0.6, 1.0]
    res = phipm_simul_iom2(PhiTask(A=A, v=v, rho=rho, tol=1e-8))
    ref = engine_run(A, v, rho, tol=1e-8)
    assert (res.substeps, res.rejections, res.matvecs, res.m_final) == \
        (ref.substeps, ref.rejections, ref.matvecs, ref.m_final)
    assert rel(res.W, ref.W) <= 1e-9


def test_swe_engine_call_matches_oracle(c0):
    ops, u0, _ = c0
    dt = 3600.0
    f = swe_rhs(ops, u0)
    J = swe_jacobian(ops, u0)
    op = OracleOperator(lambda x: dt * J.matvec(x), J.n_rows, J.nnz)
    v = [np.zeros_like(u0), dt * f]
    ref = engine_run(op, v, [0.75], tol=1e-8, trace=True)
    A = gswe.assemble_jacobian(ops, u0).scaled(dt)
    res = phipm_simul_iom2(PhiTask(A=A, v=v, rho=[0.75], tol=1e-8, trace=True))
    assert [r[3] for r in res.trace] == [r[3] for r in ref.trace]
    assert (res.substeps, res.rejections, res.matvecs, res.m_final) == \
        (ref.substeps, ref.rejections, ref.matvecs, ref.m_final)
    assert rel(res.W, ref.W) <= 1e-11


@pytest.mark.parametrize("scheme", ["exprb42", "pexprb43", "exprb53", "epi3"])
def test_c0_steps_match_oracle(c0, scheme):
    ops, u0, spec = c0
    nsteps = 3
    ref_u, ref_steps, _, log = integrate_oracle(swe_problem(ops), scheme, u0,
                                                spec.dt, nsteps * spec.dt, tol=spec.tol)
    recs = integrate(gpu_problem(ops), scheme, u0, spec.dt, nsteps * spec.dt,
                     tol=spec.tol)
    got = [(r.matvecs, r.substeps) for r in recs[1:]]
    assert got == ref_steps
    assert rel(recs[-1].u, ref_u) <= 1e-9
