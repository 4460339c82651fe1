"""SWE operator-level API on the GPU: errors, seeds, nnz at other states."""

import numpy as np
import pytest

from oracle import swe_jacobian, swe_rhs
from paper_1805_02144_b200 import swe as gswe
from paper_1805_02144_b200.integrators import EngineSeeds, step_epi3, step_exprb42, swe_problem
from paper_1805_02144_b200.states import make_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c0():
    return make_config("C0")


def test_nonfinite_state_raises(c0):
    ops, u0, _ = c0
    u = u0.copy()
    u[17] = np.nan
    with pytest.raises(ValueError):
        gswe.rhs(ops, u)
    ctx = gswe.SweContext(ops)
    ctx.set_state(u)
    with pytest.raises(ValueError):
        ctx.step("exprb42", 3600.0, 1e-8)


def test_rest_state_is_steady(c0):
    ops, _, _ = c0
    N = ops.n_g
    u = np.concatenate([np.zeros(3 * N), np.full(N, 8000.0)])
    assert np.abs(gswe.rhs(ops, u)).max() <= 1e-10 * 9.8 * 8000


def test_nnz_at_perturbed_states(c0):
    ops, u0, _ = c0
    rng = np.random.default_rng(9)
    for k in range(3):
        u = u0 + (rng.standard_normal(u0.shape) if k else 0.0)
        assert gswe.jacobian_nnz(ops, u) == swe_jacobian(ops, u).nnz


def test_seeds_roundtrip_and_step_api(c0):
    ops, u0, spec = c0
    prob = swe_problem(ops)
    seeds = EngineSeeds()
    u1 = step_exprb42(prob, u0, spec.dt, tol=spec.tol, seeds=seeds)
    assert seeds.get("exprb42/1")[1] > 1 and seeds.get("exprb42/2")[1] > 1
    u2 = step_epi3(prob, u1, u0, spec.dt, tol=spec.tol, seeds=seeds)
    assert np.isfinite(u2).all()
    with pytest.raises(ValueError):
        step_epi3(prob, u1, None, spec.dt)


def test_rhs_on_planar_reference_style_operators():
    """The C ABI takes any DiscreteOperators: a doubly periodic planar grid
    built like the reference's factory (swe.py:88-121) runs unchanged."""
    import scipy.sparse as sp
    from paper_1805_02144_b200.grid import DiscreteOperators
    from paper_1805_02144_b200.sparse import SparseMatrix
    nx = ny = 16
    dx = 1.0e5
    e = np.ones(nx) / (2 * dx)
    D1 = sp.diags([e[:-1], -e[:-1]], [1, -1], shape=(nx, nx), format="lil")
    D1[0, nx - 1] = -1 / (2 * dx)
    D1[nx - 1, 0] = 1 / (2 * dx)
    S1 = sp.diags([np.ones(nx - 1), -2 * np.ones(nx), np.ones(nx - 1)], [1, 0, -1],
                  shape=(nx, nx), format="lil") / dx ** 2
    S1[0, nx - 1] = 1 / dx ** 2
    S1[nx - 1, 0] = 1 / dx ** 2
    I = sp.identity(nx, format="csr")
    ddx = sp.kron(I, sp.csr_matrix(D1), format="csr")
    ddy = sp.kron(sp.csr_matrix(D1), I, format="csr")
    lap = (sp.kron(I, sp.csr_matrix(S1)) + sp.kron(sp.csr_matrix(S1), I)).tocsr()
    n = nx * ny
    z = sp.csr_matrix((n, n))
    nu = 0.04e-2 * dx ** 4 / 240.0
    ops = DiscreteOperators(
        Gx=SparseMatrix(ddx), Gy=SparseMatrix(ddy), Gz=SparseMatrix(z),
        Dx=SparseMatrix(ddx), Dy=SparseMatrix(ddy), Dz=SparseMatrix(z),
        Vx=SparseMatrix(-ddy), Vy=SparseMatrix(ddx), Vz=SparseMatrix(z),
        L=SparseMatrix(lap), Df=SparseMatrix(-nu * (lap @ lap)),
        n_x=np.zeros(n), n_y=np.zeros(n), n_z=np.ones(n), f=np.full(n, 1e-4),
        h_s=np.zeros(n), g=9.80616, nu=nu, n_g=n, cell_area=dx * dx)
    rng = np.random.default_rng(43)
    u = np.concatenate([5 * rng.standard_normal(2 * n), np.zeros(n),
                        8000 + 50 * rng.standard_normal(n)])
    ref = swe_rhs(ops, u)
    assert np.linalg.norm(gswe.rhs(ops, u) - ref) <= 1e-12 * np.linalg.norm(ref)
    v = rng.standard_normal(4 * n)
    J = swe_jacobian(ops, u)
    assert np.linalg.norm(gswe.assemble_jacobian(ops, u).matvec(v) - J.matvec(v)) <= \
        1e-12 * np.linalg.norm(J.matvec(v))
    assert gswe.jacobian_nnz(ops, u) == J.nnz


def test_diagnostics_match_reference_formula(c0):
    """swe.py:226-237 restated: mass/energy/enstrophy with the scalar
    cell_area, and the per-cell-area variant."""
    ops, u0, _ = c0
    N = ops.n_g
    ux, uy, uz, h = np.split(u0, 4)
    zeta = ops.Vx.csr @ ux + ops.Vy.csr @ uy + ops.Vz.csr @ uz
    for weighted in (False, True):
        w = ops.areas if weighted else np.full(N, ops.cell_area)
        mass = np.sum(w * h)
        energy = np.sum(w * (ops.g * h + 0.5 * (ux * ux + uy * uy + uz * uz)))
        ens = np.sum(w * (zeta + ops.f) ** 2 / (2.0 * h))
        d = gswe.diagnostics(ops, u0, area_weighted=weighted)
        assert abs(d.mass - mass) <= 1e-13 * mass
        assert abs(d.energy - energy) <= 1e-13 * energy
        assert abs(d.enstrophy - ens) <= 1e-12 * ens
    bad = u0.copy()
    bad[3 * N + 5] = -1.0
    with pytest.raises(ValueError):
        gswe.diagnostics(ops, bad)


def test_mass_conserved_by_steps(c0):
    """Flux-form divergence: area-weighted mass is conserved to rounding by
    every scheme over several steps (acceptance criterion 8 analogue,
    test_acceptance.py:154-168), measured on the resident state."""
    ops, u0, spec = c0
    ctx = gswe.SweContext(ops)
    ctx.set_state(u0)
    d0 = gswe.diagnostics(ops, u0, area_weighted=True)
    for k in range(6):
        ctx.step("exprb42", spec.dt, spec.tol)
    u = ctx.get_state()
    d = gswe.diagnostics(ops, u, area_weighted=True)
    dm, de, dz = d.drifts(d0)
    assert abs(dm) <= 1e-12
    assert abs(de) <= 1e-3 and abs(dz) <= 1e-2
