"""Sphere grid and configuration states (CPU)."""

import numpy as np
import pytest

from paper_1805_02144_b200.grid import (EARTH_RADIUS, hilbert_keys, mesh_geometry,
                                        n_cells, sphere_operators)
from paper_1805_02144_b200.states import CONFIGS, make_config


@pytest.fixture(scope="module", params=[2, 4])
def ops(request):
    return sphere_operators(request.param)


def test_counts_and_areas(ops):
    assert ops.n_g == n_cells(ops.level)
    assert abs(ops.areas.sum() / (4 * np.pi * EARTH_RADIUS ** 2) - 1) < 1e-13
    assert set(np.unique(ops.mesh.deg)) == {5, 6}
    assert (ops.mesh.deg == 5).sum() == 12


def test_neighbours_symmetric(ops):
    m = ops.mesh
    pairs = {(i, int(j)) for i in range(ops.n_g) for j in m.nbr[i] if j >= 0}
    assert all((j, i) in pairs for i, j in pairs)


def test_row_sums_vanish(ops):
    one = np.ones(ops.n_g)
    for name in ("Gx", "Gy", "Gz", "Vx", "Vy", "Vz", "L"):
        M = getattr(ops, name).csr
        assert np.abs(M @ one).max() <= 1e-12 * np.abs(M).max()


def test_divergence_conserves_mass(ops):
    rng = np.random.default_rng(0)
    F = rng.standard_normal((3, ops.n_g))
    div = ops.Dx.matvec(F[0]) + ops.Dy.matvec(F[1]) + ops.Dz.matvec(F[2])
    assert abs((ops.areas * div).sum()) <= 1e-13 * np.abs(ops.areas * div).sum()


def test_operators_consistent():
    errs = []
    for L in (4, 5):
        ops = sphere_operators(L)
        x = ops.mesh.x
        c = np.array([0.3, -0.5, 0.8])
        e = (x @ c) * EARTH_RADIUS
        ct = c - x * (x @ c)[:, None]
        g = np.stack([ops.Gx.matvec(e), ops.Gy.matvec(e), ops.Gz.matvec(e)], 1)
        lap = ops.L.matvec(e)
        errs.append((np.abs(g - ct).max(),
                     np.abs(lap + 2 * e / EARTH_RADIUS ** 2).max() * EARTH_RADIUS ** 2 / 2))
    # both converge (first order in max norm on the non-optimised mesh)
    assert errs[1][0] < 0.6 * errs[0][0]
    assert errs[1][1] < 0.6 * errs[0][1]


def test_df_is_minus_nu_L_squared(ops):
    D = (-ops.nu * (ops.L.csr @ ops.L.csr)).tocsr()
    assert abs(D - ops.Df.csr).max() == 0.0


def test_hilbert_order_is_local():
    ops = sphere_operators(5)
    m = ops.mesh
    d = np.abs(m.nbr - np.arange(ops.n_g)[:, None])[m.nbr >= 0]
    assert np.median(d) < 0.01 * ops.n_g


def test_hilbert_keys_distinct():
    rng = np.random.default_rng(1)
    p = rng.uniform(-1, 1, (1000, 3))
    assert len(np.unique(hilbert_keys(p))) == 1000


@pytest.mark.parametrize("name", ["C0", "C1", "C2"])
def test_config_states(name):
    ops, u0, spec = make_config(name, level=3)
    N = ops.n_g
    ux, uy, uz, h = np.split(u0, 4)
    x = ops.mesh.x
    assert np.abs(ux * x[:, 0] + uy * x[:, 1] + uz * x[:, 2]).max() < 1e-9
    assert h.min() > 1000.0
    assert np.isfinite(u0).all()
    if name == "C2":
        assert ops.h_s.max() > 500.0


def test_config3_jet():
    ops, u0, spec = make_config("C3", level=4)
    ux, uy, uz, h = np.split(u0, 4)
    speed = np.sqrt(ux ** 2 + uy ** 2 + uz ** 2)
    assert 40.0 < speed.max() <= 60.0 + 1e-9
    assert abs(np.average(h, weights=ops.areas) - 10000.0) < 50.0


def test_configs_table():
    assert CONFIGS["C3"].level == 8 and CONFIGS["C3"].dt == 600.0
    assert CONFIGS["C0"].steps == 24 and CONFIGS["C0"].tol == 1e-8
