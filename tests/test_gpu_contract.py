"""API contract of the GPU path against the reference semantics, and the
device branches the config runs do not reach (all against the oracle port):

* ``seeds=None`` starts every engine call cold (integrators.py:128), also
  after earlier calls on the same cached device context;
* a ``DiscreteOperators`` whose Df is not -nu L@L is rejected (the device
  applies Df as -nu L(L .)), one whose Df is is accepted;
* the dense phi phase beyond shared memory (augmented dimension >= 69, the
  global-scratch branch) in the generic engine, in the SWE engine entry and in
  the split step's dense kernel, up to the dense cap (dim 256) and past it
  (ValueError, kernels.py:159-163);
* m_max above 100 on the SWE operator (the basis grows);
* the explicit-orthogonalisation fallback and a happy breakdown inside the
  tiled IOM2 sweep;
* the non-tiled step path (operators outside the compact difference form);
* an unbounded trace (more attempts than the first trace buffer holds).
"""

import ctypes as C
import dataclasses

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import engine_run, integrate_oracle, step_oracle, swe_problem
from oracle.expint_oracle import CallLog, OracleOperator, OracleSeeds
from oracle.swe_oracle import swe_jacobian
from paper_1805_02144_b200 import _native as nat
from paper_1805_02144_b200 import swe as gswe
from paper_1805_02144_b200.integrators import _StepStats, step_exprb42, swe_problem as gprob
from paper_1805_02144_b200.phipm import PhiTask, phipm_simul_iom2
from paper_1805_02144_b200.sparse import SparseMatrix
from paper_1805_02144_b200.states import make_config

pytestmark = pytest.mark.gpu
TOL = 1e-9


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def oracle_run(op, task):
    t = dict(task)
    return engine_run(op, t.pop("v"), t.pop("rho"), trace=True, **t)


def counters(r):
    return (r.substeps, r.rejections, r.matvecs, r.m_final)


# ------------------------------------------------------------------ seeds

def test_step_without_seeds_is_cold_every_call():
    """Three step_exprb42(prob, u, dt) calls with seeds=None, after an
    integrate() warmed the cached context: each equals the oracle run with
    fresh (None, 1) seeds."""
    from paper_1805_02144_b200.integrators import integrate
    ops, u0, spec = make_config("C0")
    prob = gprob(ops)
    integrate(prob, "exprb42", u0, spec.dt, 3 * spec.dt, tol=spec.tol)  # warms the seeds
    u = u0
    for k in range(3):
        log = CallLog()
        ref = step_oracle(swe_problem(ops), "exprb42", u, spec.dt, spec.tol, OracleSeeds(), log)
        st = _StepStats()
        got = step_exprb42(prob, u, spec.dt, tol=spec.tol, stats=st)
        assert (st.matvecs, st.substeps) == (sum(c[3] for c in log.calls),
                                             sum(c[1] for c in log.calls)), k
        assert rel(got, ref) <= TOL
        u = ref


# --------------------------------------------------------------------- Df

def test_df_other_than_minus_nu_LL_is_rejected():
    ops, u0, _ = make_config("C0")
    bad = dataclasses.replace(ops, Df=SparseMatrix(2.0 * ops.Df.csr))
    with pytest.raises(ValueError, match="Df"):
        gswe.SweContext(bad)
    perturbed = ops.Df.csr.copy()
    perturbed.data[7] *= 1.0 + 1e-6
    with pytest.raises(ValueError, match="Df"):
        gswe.SweContext(dataclasses.replace(ops, Df=SparseMatrix(perturbed)))
    # an explicit zero outside L@L's pattern is harmless; a nonzero is not
    extra = ops.Df.csr.tolil()
    far = int(np.argmax(np.abs(ops.n_z - ops.n_z[0])))
    extra[0, far] = 1e-30
    with pytest.raises(ValueError, match="Df"):
        gswe.SweContext(dataclasses.replace(ops, Df=SparseMatrix(extra.tocsr())))


def test_df_recomputed_product_is_accepted():
    """Df assembled in another summation order (L.T.T @ L) passes the check."""
    ops, u0, _ = make_config("C0")
    L = ops.L.csr
    df = (-ops.nu) * (sp.csr_matrix(L.T).T.tocsr() @ L)
    ctx = gswe.SweContext(dataclasses.replace(ops, Df=SparseMatrix(df.tocsr())))
    assert np.all(np.isfinite(ctx.rhs(u0)))


# ---------------------------------------------------------- dense phi cap

def _stiff(n, seed, lo=0.0, hi=2.0):
    rng = np.random.default_rng(seed)
    Q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    A = Q @ np.diag(-np.logspace(lo, hi, n)) @ Q.T
    return A, rng


@pytest.mark.parametrize("m,p", [(100, 4), (180, 2), (252, 3)])
def test_generic_engine_dense_global_scratch(m, p):
    """dim = m + p + 1 in {105, 183, 256}: the dense phase runs on the global
    scratch (kDenseSmem holds dim <= 46 in the cooperative kernel)."""
    n = 400
    A, rng = _stiff(n, 5 + m)
    v = [rng.standard_normal(n) for _ in range(p + 1)]
    task = dict(v=v, rho=[1.0], tol=1e-12, m_init=m, m_max=m)
    r = phipm_simul_iom2(PhiTask(A=SparseMatrix.from_dense(A), trace=True, **task))
    o = oracle_run(A, task)
    assert counters(r) == counters(o)
    assert [t[3] for t in r.trace] == [t[3] for t in o.trace]
    assert max(t[3] for t in r.trace) + p + 1 >= 69
    assert rel(r.W, o.W) <= TOL


def test_dense_cap_exceeded_raises_like_reference():
    n = 400
    A, rng = _stiff(n, 3)
    v = [rng.standard_normal(n) for _ in range(4)]
    task = dict(v=v, rho=[1.0], tol=1e-12, m_init=253, m_max=253)
    with pytest.raises(ValueError, match="exceeds cap 256"):
        oracle_run(A, task)
    with pytest.raises(ValueError, match="exceeds cap 256"):
        phipm_simul_iom2(PhiTask(A=SparseMatrix.from_dense(A), **task))


def test_swe_engine_m100_and_beyond():
    """The SWE operator (tiled IOM2 sweep) at m = 100 (dim 103) and, with
    m_max = 140 > the context's 100, at m = 140: the basis grows."""
    ops, u0, spec = make_config("C0")
    J = gswe.assemble_jacobian(ops, u0).scaled(spec.dt)
    rng = np.random.default_rng(3)
    fn = gswe.rhs(ops, u0)
    v = [np.zeros_like(u0), spec.dt * fn, 1e-3 * spec.dt * rng.standard_normal(u0.shape[0])]
    Jo = swe_jacobian(ops, u0)
    op = OracleOperator(lambda x: spec.dt * Jo.matvec(x), Jo.n_rows, Jo.nnz)
    for m in (100, 140):
        task = dict(v=v, rho=[0.5, 1.0], tol=1e-10, m_init=m, m_max=m)
        r = phipm_simul_iom2(PhiTask(A=J, trace=True, **task))
        op.count = 0
        o = oracle_run(op, task)
        assert counters(r) == counters(o), m
        assert [t[3] for t in r.trace] == [t[3] for t in o.trace]
        assert rel(r.W, o.W) <= TOL


def test_step_dense_kernel_global_scratch():
    """The split step's k_swe_dense beyond shared memory: the first engine
    call of an exprb42 step forced to start at m = 100 (seeds)."""
    ops, u0, spec = make_config("C0")
    ctx = gswe.SweContext(ops)
    ctx.set_state(u0)
    ctx.reset_seeds()
    ctx.set_seeds("exprb42/1", None, 100)
    ctx.set_seeds("exprb42/2", None, 90)
    cs = ctx.step("exprb42", spec.dt, spec.tol)
    seeds = OracleSeeds()
    seeds.table["exprb42/1"] = (None, 100)
    seeds.table["exprb42/2"] = (None, 90)
    log = CallLog()
    ref = step_oracle(swe_problem(ops), "exprb42", u0, spec.dt, spec.tol, seeds, log)
    assert [(c.substeps, c.rejections, c.matvecs, c.m_final) for c in cs] == \
        [tuple(c[1:5]) for c in log.calls]
    assert rel(ctx.get_state(), ref) <= TOL


# ------------------------------------------- IOM2 fallback and breakdown

def _explicit(ctx):
    return int(nat.load().eik_swe_explicit_orth(ctx.h))


def test_tiled_sweep_breakdown_and_explicit_orthogonalisation():
    """At rest over a flat depth a constant height perturbation is in the
    kernel of J (G, D, L rows sum to zero): z = J v_0 = 0, the Gram-identity
    norm is rejected (explicit pass) and the sweep breaks down at j = 0."""
    ops, _, _ = make_config("C0")
    n = ops.n_g
    u = np.concatenate([np.zeros(3 * n), np.full(n, 5000.0)])
    ctx = gswe.context(ops)
    before = _explicit(ctx)
    J = gswe.assemble_jacobian(ops, u).scaled(600.0)
    v = [np.zeros(4 * n), np.concatenate([np.zeros(3 * n), np.ones(n)])]
    r = phipm_simul_iom2(PhiTask(A=J, v=v, rho=[1.0], tol=1e-8, m_init=8, trace=True))
    assert _explicit(ctx) > before
    Jo = swe_jacobian(ops, u)
    o = engine_run(OracleOperator(lambda x: 600.0 * Jo.matvec(x), Jo.n_rows, Jo.nnz),
                   v, [1.0], tol=1e-8, m_init=8, trace=True)
    assert counters(r) == counters(o)
    assert rel(r.W, o.W) <= TOL


def test_explicit_orthogonalisation_inside_steps_counted():
    """The counter the fallback test reads is live in normal steps too (it
    only grows; no step of C0 needs the fallback)."""
    ops, u0, spec = make_config("C0")
    ctx = gswe.SweContext(ops)
    ctx.set_state(u0)
    e0 = _explicit(ctx)
    ctx.step("exprb42", spec.dt, spec.tol)
    assert _explicit(ctx) >= e0


# ------------------------------------------------------ non-tiled path

def _info(ctx):
    out = (C.c_int64 * 16)()
    nat.check(nat.load().eik_swe_info(ctx.h, out), "info")
    return list(out)


def test_non_tiled_step_path_matches_oracle():
    """Operators outside the compact difference form (G rows that do not sum
    to zero) run the generic per-matvec path; whole steps against the oracle."""
    from test_gpu_planar_steps import planar_ops, smooth_state
    ops = planar_ops()
    dx = 1.0e5
    n = ops.n_g
    gx = (ops.Gx.csr + sp.identity(n, format="csr") * (1e-3 / dx)).tocsr()
    ops = dataclasses.replace(ops, Gx=SparseMatrix(gx))
    u0 = smooth_state(ops)
    ctx = gswe.SweContext(ops)
    assert _info(ctx)[7] == 0  # compact stencil invalid -> non-tiled path
    ctx.set_state(u0)
    ctx.reset_seeds()
    steps = []
    for _ in range(2):
        cs = ctx.step("exprb42", 900.0, 1e-8)
        steps.append((sum(c.matvecs for c in cs), sum(c.substeps for c in cs)))
    ref, ref_steps, _, _ = integrate_oracle(swe_problem(ops), "exprb42", u0, 900.0, 1800.0,
                                            tol=1e-8)
    assert steps == ref_steps
    assert rel(ctx.get_state(), ref) <= TOL


# -------------------------------------------------------------- trace

def test_trace_is_unbounded():
    """m_max = 3 forces tiny substeps: ~12k attempts, three times the first
    4096-row trace buffer.  The device trace is complete (one row per
    attempt, numbered 1..N) and equals the oracle's row for row well past
    row 4096.  (Over 12k chaotic accept/reject decisions a rounding-level
    difference in eps eventually flips one, so the comparison is over the
    common prefix, which must extend beyond the first buffer.)"""
    n = 30
    A, rng = _stiff(n, 11, 0.0, 3.0)
    v = [rng.standard_normal(n), rng.standard_normal(n)]
    task = dict(v=v, rho=[1.0], tol=1e-8, m_init=1, m_max=3)
    o = oracle_run(A, task)
    r = phipm_simul_iom2(PhiTask(A=SparseMatrix.from_dense(A), trace=True, **task))
    assert len(r.trace) == r.substeps + r.rejections > 4096
    assert [t[0] for t in r.trace] == list(range(1, len(r.trace) + 1))
    same = 0
    for a, b in zip(r.trace, o.trace):
        if (a[3], a[6]) != (b[3], b[6]) or abs(a[2] - b[2]) > 1e-9 * b[2]:
            break
        same += 1
    assert same > 2 * 4096, same
