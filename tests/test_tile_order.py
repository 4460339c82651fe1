"""Device cell order (eik_tile_order, host-only C ABI): the recursive
coordinate bisection that eik_swe_create uses to cut the grid into the
Krylov pass's tiles -- a permutation, equal leaves, compact halos."""

import ctypes as C

import numpy as np
import pytest

from paper_1805_02144_b200 import _native as nat
from paper_1805_02144_b200.grid import cached_sphere_operators


def tile_order(px, py, pz, ntiles):
    n = len(px)
    ord_ = np.empty(n, dtype=np.int32)
    starts = np.empty(ntiles + 1, dtype=np.int32)
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (px, py, pz)]
    nat.check(nat.load().eik_tile_order(n, *(nat.dptr(a) for a in arrs), ntiles,
                                        ord_.ctypes.data_as(C.POINTER(C.c_int32)),
                                        starts.ctypes.data_as(C.POINTER(C.c_int32))),
              "tile_order")
    return ord_, starts


def halo_ratios(csr, ord_, starts):
    """(E1 cells, E2 cells) summed over tiles, per own cell."""
    ip, ix = csr.indptr, csr.indices
    n = len(ord_)
    s1 = s2 = 0
    for t in range(len(starts) - 1):
        own = ord_[starts[t]:starts[t + 1]]
        e1 = set(own.tolist())
        for i in own:
            e1.update(ix[ip[i]:ip[i + 1]].tolist())
        e2 = set(e1)
        for i in e1.difference(own.tolist()):
            e2.update(ix[ip[i]:ip[i + 1]].tolist())
        s1 += len(e1)
        s2 += len(e2)
    return s1 / n, s2 / n


@pytest.fixture(scope="module")
def l5():
    return cached_sphere_operators(5)


@pytest.mark.parametrize("ntiles", [1, 7, 40, 64])
def test_permutation_and_equal_leaves(l5, ntiles):
    ord_, starts = tile_order(l5.n_x, l5.n_y, l5.n_z, ntiles)
    n = l5.n_g
    assert np.array_equal(np.sort(ord_), np.arange(n))
    assert starts[0] == 0 and starts[-1] == n
    sizes = np.diff(starts)
    assert sizes.min() >= 0 and sizes.max() - sizes.min() <= 1
    # each leaf is kept in user (grid) order
    for t in range(ntiles):
        leaf = ord_[starts[t]:starts[t + 1]]
        assert np.all(np.diff(leaf) > 0)


def test_deterministic(l5):
    a = tile_order(l5.n_x, l5.n_y, l5.n_z, 40)
    b = tile_order(l5.n_x, l5.n_y, l5.n_z, 40)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_tiles_more_compact_than_index_ranges(l5):
    """Same tile count and sizes, halos smaller than contiguous ranges of the
    grid's own (Hilbert) order -- the point of the device order."""
    nt = 40
    ord_, starts = tile_order(l5.n_x, l5.n_y, l5.n_z, nt)
    e1, e2 = halo_ratios(l5.L.csr, ord_, starts)
    ident = np.arange(l5.n_g, dtype=np.int32)
    e1h, e2h = halo_ratios(l5.L.csr, ident, starts)
    assert e1 < e1h and e2 < e2h
    assert e2 < 1.9


def test_constant_positions_keep_index_order():
    """The reference's planar operators have n = (0, 0, 1) everywhere."""
    n = 1000
    ord_, starts = tile_order(np.zeros(n), np.zeros(n), np.ones(n), 9)
    assert np.array_equal(ord_, np.arange(n))
    assert np.all(np.diff(starts) >= 111)


def test_more_tiles_than_cells():
    ord_, starts = tile_order(np.arange(3.0), np.zeros(3), np.zeros(3), 5)
    assert sorted(ord_.tolist()) == [0, 1, 2]
    assert starts[-1] == 3 and np.all(np.diff(starts) >= 0)


def test_invalid_arguments():
    with pytest.raises(ValueError):
        tile_order(np.zeros(4), np.zeros(4), np.zeros(4), 0)
