"""The reference's engine/integrator test suite (pkg/tests/test_phipm.py,
test_integrators.py, test_acceptance.py) restated against the GPU engine."""

import math

import numpy as np
import pytest
from scipy.linalg import expm

import paper_1805_02144_b200.phipm as phipm_mod
from oracle import engine_run
from paper_1805_02144_b200 import SparseMatrix
from paper_1805_02144_b200.integrators import SCHEME_NAMES, SemilinearProblem, integrate
from paper_1805_02144_b200.phipm import (MatvecOperator, PhiTask, PhipmFailure,
                                         phipm_simul_iom2)

pytestmark = pytest.mark.gpu


def phi_dense_all(Z, kmax):
    """[phi_0(Z), ..., phi_kmax(Z)] from one block-augmented exponential."""
    n = Z.shape[0]
    big = np.zeros((n * (kmax + 1), n * (kmax + 1)))
    big[:n, :n] = Z
    for j in range(kmax):
        big[n * j:n * (j + 1), n * (j + 1):n * (j + 2)] = np.eye(n)
    E = expm(big)
    return [E[:n, j * n:(j + 1) * n] for j in range(kmax + 1)]


def dense_combination(A, v, rho):
    p = len(v) - 1
    out = np.zeros((v[0].shape[0], len(rho)))
    for i, r in enumerate(rho):
        phis = phi_dense_all(r * np.asarray(A), p)
        acc = np.zeros_like(v[0])
        for ell in range(p + 1):
            acc = acc + r ** ell * (phis[ell] @ v[ell])
        out[:, i] = acc
    return out


@pytest.fixture
def stiff_system():
    rng = np.random.default_rng(23)
    n = 40
    Q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    A = Q @ np.diag(-np.logspace(0, 3, n)) @ Q.T
    v = [rng.standard_normal(n) for _ in range(4)]
    return A, v


def test_engine_matches_dense_oracle(stiff_system):
    A, v = stiff_system
    rho = [0.25, 0.6, 1.0]
    res = phipm_simul_iom2(PhiTask(A=A, v=v, rho=rho, tol=1e-8))
    ref = dense_combination(A, v, rho)
    for i in range(len(rho)):
        assert np.max(np.abs(res.W[:, i] - ref[:, i])) / np.max(np.abs(ref)) <= 100 * 1e-8


def test_engine_counters_match_oracle(stiff_system):
    A, v = stiff_system
    for rho in ([0.25, 0.6, 1.0], [0.123456, 0.654321, 1.0], [1.0]):
        r = phipm_simul_iom2(PhiTask(A=A, v=v, rho=rho, tol=1e-8, trace=True))
        o = engine_run(A, v, rho, tol=1e-8, trace=True)
        assert (r.substeps, r.rejections, r.matvecs, r.m_final) == \
            (o.substeps, o.rejections, o.matvecs, o.m_final)
        assert [t[3] for t in r.trace] == [t[3] for t in o.trace]
        # the stiff (|A| = 1e3) full-dimension solve amplifies rounding through
        # 8 squarings: engine accuracy is 100 * tol (test_phipm.py:47-56)
        assert np.linalg.norm(r.W - o.W) <= 1e-6 * np.linalg.norm(o.W)


def test_tighter_tolerance_is_more_accurate(stiff_system):
    A, v = stiff_system
    ref = dense_combination(A, v, [1.0])[:, 0]
    errs = []
    for tol in (1e-4, 1e-8):
        res = phipm_simul_iom2(PhiTask(A=A, v=v, rho=[1.0], tol=tol))
        errs.append(np.max(np.abs(res.W[:, 0] - ref)) / np.max(np.abs(ref)))
    assert errs[1] <= errs[0] and errs[0] <= 1e-2 and errs[1] <= 1e-6


def test_zero_skip_reduces_matvecs(stiff_system):
    A, v = stiff_system
    n = A.shape[0]
    v = [np.zeros(n), np.zeros(n), v[2], v[3]]
    on = phipm_simul_iom2(PhiTask(A=A, v=v, rho=[1.0], tol=1e-6, zero_skip=True))
    off = phipm_simul_iom2(PhiTask(A=A, v=v, rho=[1.0], tol=1e-6, zero_skip=False))
    assert on.matvecs < off.matvecs
    assert np.max(np.abs(on.W - off.W)) <= 1e-13 * max(1.0, np.max(np.abs(off.W)))


def test_outputs_hit_rho_exactly(stiff_system):
    A, v = stiff_system
    rho = [0.123456, 0.654321, 1.0]
    res = phipm_simul_iom2(PhiTask(A=A, v=v, rho=rho, tol=1e-8))
    ref = dense_combination(A, v, rho)
    assert np.max(np.abs(res.W - ref)) <= 1e-5 * np.max(np.abs(ref))


def test_trace_csv(tmp_path, stiff_system):
    A, v = stiff_system
    res = phipm_simul_iom2(PhiTask(A=A, v=v, rho=[1.0], tol=1e-6, trace=True))
    assert len(res.trace) >= res.substeps
    path = tmp_path / "trace.csv"
    res.write_trace_csv(path)
    lines = path.read_text().strip().splitlines()
    assert lines[0].startswith("attempt,") and len(lines) == len(res.trace) + 1


def test_failure_carries_diagnostics(monkeypatch, stiff_system):
    A, v = stiff_system
    monkeypatch.setattr(phipm_mod, "MAX_SUBSTEPS", 1)
    with pytest.raises(PhipmFailure) as exc:
        phipm_simul_iom2(PhiTask(A=A, v=v, rho=[1.0], tol=1e-13))
    err = exc.value
    assert err.t_reached < 1.0
    assert err.substeps + err.rejections <= 1
    assert err.matvecs >= 0


def test_full_dimension_generic_mgs():
    # m reaches n: iom = n (full orthogonalisation, krylov.py / phipm.py:207-209)
    rng = np.random.default_rng(13)
    n = 12
    A = rng.standard_normal((n, n)) - 5 * np.eye(n)
    v = [np.zeros(n), rng.standard_normal(n)]
    res = phipm_simul_iom2(PhiTask(A=A, v=v, rho=[1.0], tol=1e-12, m_init=12))
    ref = dense_combination(A, v, [1.0])
    assert np.max(np.abs(res.W - ref)) <= 1e-9 * np.max(np.abs(ref))


def test_engine_accepts_sparse_and_operator_inputs(stiff_system):
    """test_phipm.py:73-82: SparseMatrix, scipy CSR and a MatvecOperator
    around a host callable (device engine, one host round trip per matvec)."""
    import scipy.sparse as sp
    A, v = stiff_system
    ref = phipm_simul_iom2(PhiTask(A=A, v=v, rho=[1.0], tol=1e-8)).W
    for wrapped in (SparseMatrix.from_dense(A), sp.csr_matrix(A),
                    MatvecOperator(lambda x: A @ x, A.shape[0], A.size)):
        res = phipm_simul_iom2(PhiTask(A=wrapped, v=v, rho=[1.0], tol=1e-8))
        assert np.allclose(res.W, ref, rtol=1e-6, atol=1e-10)


def test_callable_operator_matches_oracle(stiff_system):
    """The host-callback route: the callable is invoked exactly once per
    performed matvec (the reference's _CountingOperator count), counters and
    trace equal the oracle's, W within 1e-9."""
    from oracle.expint_oracle import OracleOperator
    A, v = stiff_system
    seen = []

    def mv(x):
        seen.append(x.copy())
        return A @ x

    for rho in ([1.0], [0.3, 0.7, 1.0]):
        seen.clear()
        r = phipm_simul_iom2(PhiTask(A=MatvecOperator(mv, 40, A.size), v=v, rho=rho,
                                     tol=1e-8, trace=True))
        o = engine_run(OracleOperator(lambda x: A @ x, 40, A.size), v, rho, tol=1e-8,
                       trace=True)
        assert len(seen) == r.matvecs
        assert (r.substeps, r.rejections, r.matvecs, r.m_final) == \
            (o.substeps, o.rejections, o.matvecs, o.m_final)
        assert [t[3] for t in r.trace] == [t[3] for t in o.trace]
        # same bound as test_engine_counters_match_oracle on this fixture: the
        # full-dimension (m = n = 40) stiff solve amplifies rounding
        assert np.linalg.norm(r.W - o.W) <= 1e-6 * np.linalg.norm(o.W)


def test_callable_operator_repeated_calls_are_identical(stiff_system):
    """The host-callback route is deterministic: 25 calls (interleaved with
    device CSR calls on other sizes) give bitwise-identical W and counters."""
    A, v = stiff_system
    first = None
    rng = np.random.default_rng(4)
    B = rng.standard_normal((64, 64)) - 8.0 * np.eye(64)
    vb = [rng.standard_normal(64)]
    for k in range(25):
        r = phipm_simul_iom2(PhiTask(A=MatvecOperator(lambda x: A @ x, 40, A.size), v=v,
                                     rho=[0.5, 1.0], tol=1e-8))
        key = (r.W.tobytes(), r.substeps, r.rejections, r.matvecs, r.m_final)
        first = first or key
        assert key == first, k
        phipm_simul_iom2(PhiTask(A=B, v=vb, rho=[1.0], tol=1e-8))


def test_callable_operator_exception_propagates(stiff_system):
    A, v = stiff_system
    calls = []

    def bad(x):
        calls.append(1)
        if len(calls) == 3:
            raise ZeroDivisionError("boom")
        return A @ x

    with pytest.raises(ZeroDivisionError):
        phipm_simul_iom2(PhiTask(A=MatvecOperator(bad, 40, A.size), v=v, rho=[1.0],
                                 tol=1e-8))
    assert len(calls) == 3  # no further requests after the failure
    # the context is reusable afterwards
    r = phipm_simul_iom2(PhiTask(A=MatvecOperator(lambda x: A @ x, 40, A.size), v=v,
                                 rho=[1.0], tol=1e-8))
    assert np.all(np.isfinite(r.W))


def test_context_finalised_inside_callable_is_deferred(stiff_system, monkeypatch):
    """A device context destroyed while the host-callback engine waits for the
    host (a garbage collector running inside the callable) must not touch the
    device: cudaFree would wait for the engine's kernel, which waits for the
    host.  libeik defers such destroys until the call returns; a libeik call
    from inside the callable is an error."""
    import ctypes as C
    import gc
    import scipy.sparse as sp
    from paper_1805_02144_b200 import _native as nat
    monkeypatch.setenv("EIK_CB_TIMEOUT_S", "30")
    A, v = stiff_system
    ref = phipm_simul_iom2(PhiTask(A=A, v=v, rho=[1.0], tol=1e-8))

    class Holder:
        pass

    def make_garbage():
        csr = sp.csr_matrix(A)
        view, keep = nat.csr_view(csr)
        h = C.c_void_p()
        nat.check(nat.load().eik_csr_create(40, view, 0, 40, C.byref(h)), "eik_csr_create")
        hold = Holder()
        hold.me = hold  # a reference cycle: freed by the collector only
        hold.ctx = phipm_mod._CsrCtx(h)

    gc.collect()
    gc.disable()
    try:
        make_garbage()
        calls = []

        def mv(x):
            if not calls:
                gc.collect()  # runs _CsrCtx.__del__ -> eik_csr_destroy
            calls.append(1)
            return A @ x

        r = phipm_simul_iom2(PhiTask(A=MatvecOperator(mv, 40, A.size), v=v, rho=[1.0],
                                     tol=1e-8))
    finally:
        gc.enable()
    assert (r.substeps, r.rejections, r.matvecs, r.m_final) == \
        (ref.substeps, ref.rejections, ref.matvecs, ref.m_final)
    assert np.allclose(r.W, ref.W, rtol=1e-6, atol=1e-10)

    def reentrant(x):
        phipm_simul_iom2(PhiTask(A=A, v=v, rho=[1.0], tol=1e-8))
        return A @ x

    with pytest.raises(ValueError, match="inside a matvec callback"):
        phipm_simul_iom2(PhiTask(A=MatvecOperator(reentrant, 40, A.size), v=v, rho=[1.0],
                                 tol=1e-8))


def test_callable_jacobian_in_integrator_steps():
    """A problem whose jac returns a MatvecOperator (host callable) steps
    through the device engine like the SparseMatrix one."""
    L, problem, u0 = make_linear_problem()
    hp = SemilinearProblem(n=problem.n, f=problem.f,
                           jac=lambda u: MatvecOperator(lambda x: L @ x, L.shape[0],
                                                        int(np.count_nonzero(L))))
    a = integrate(problem, "exprb42", u0, 0.25, 0.5, tol=1e-10)[-1].u
    b = integrate(hp, "exprb42", u0, 0.25, 0.5, tol=1e-10)[-1].u
    assert np.linalg.norm(a - b) <= 1e-9 * np.linalg.norm(a)


def make_linear_problem(seed=1, n=24):
    rng = np.random.default_rng(seed)
    Q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    L = Q @ np.diag(-np.logspace(-1, 2, n)) @ Q.T
    Ls = SparseMatrix.from_dense(L)
    return L, SemilinearProblem(n=n, f=lambda u: Ls.matvec(u), jac=lambda u: Ls,
                                name="linear"), rng.standard_normal(n)


@pytest.mark.parametrize("scheme", SCHEME_NAMES)
def test_linear_exactness(scheme):
    # test_integrators.py:32-40 through the GPU engine (host step route)
    L, problem, u0 = make_linear_problem()
    tol = 1e-10
    records = integrate(problem, scheme, u0, 0.25, 1.0, tol=tol)
    exact = expm(L) @ u0
    assert np.max(np.abs(records[-1].u - exact)) / np.max(np.abs(exact)) <= 100 * tol


@pytest.mark.parametrize("scheme,order", [
    ("rb_euler", 2), ("epi3", 3), ("exprb42", 4), ("pexprb43", 4), ("exprb53", 5)])
def test_empirical_order(scheme, order):
    n = 12
    lam = -np.logspace(0, 2, n)
    problem = SemilinearProblem(
        n=n, f=lambda u: lam * u + np.sin(u),
        jac=lambda u: SparseMatrix.from_dense(np.diag(lam + np.cos(u))))
    u0 = np.linspace(0.5, 1.5, n)
    ref = integrate(problem, "exprb53", u0, 1e-3, 0.5, tol=1e-12)[-1].u
    errs = [np.max(np.abs(integrate(problem, scheme, u0, dt, 0.5, tol=1e-12)[-1].u - ref))
            for dt in (0.05, 0.025)]
    assert math.log2(errs[0] / errs[1]) >= order - 0.6
