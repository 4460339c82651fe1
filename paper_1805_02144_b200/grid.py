"""Icosahedral geodesic (Voronoi) sphere grid -> ``DiscreteOperators``.

The reference ships only a doubly-periodic planar operator factory
(swe.py:88-121) and leaves the sphere as an extension point (swe.py:10-12);
the paper defers the finite-volume discretisation to [Pudykiewicz2011]
(PAPER.md:316-320).  This module is therefore new code, written so that the
reference's own ``rhs``/``assemble_jacobian`` (swe.py:149-223) run unchanged
on its output, and so that the GPU path reads exactly the same operators.

Grid: recursive bisection of the icosahedron to level ``L`` (N_g = 10*4^L+2
nodes), one Voronoi control volume per node, nodes ordered
along a 3-D Hilbert curve so that a cell's 5-6 neighbours sit close to it in
memory (the order of the reference-facing ``[u_x;u_y;u_z;h]`` layout; libeik
renumbers cells on the device into compact tiles, see eik_tile_order).

Finite-volume operators on cell i with neighbours j (Voronoi edge e_ij of arc
length l_ij, outward unit normal n_ij and counter-clockwise unit tangent t_ij
at the edge midpoint, centre distance d_ij, cell area A_i, radius a):

* gradient   G_k(i,j) = [P_i l_ij a (m_ij - x_i) / (A_i d_ij)]_k,
             G_k(i,i) = -sum_j G_k(i,j)
  (Perot reconstruction of the edge-normal differences (e_j-e_i)/d_ij from
  the edge midpoints m_ij, exact for linear fields on a planar cell;
  projected on the tangent plane P_i = I - x_i x_i^T.  The plain
  Green-Gauss form is inconsistent on a non-centroidal Voronoi mesh);
* divergence D_k(i,j) = l_ij n_ij,k / (2 A_i),         D_k(i,i) = +sum_j D_k(i,j)
  (flux form with edge average (F_i+F_j)/2: sum_i A_i div_i = 0 exactly);
* vorticity  V_k(i,j) = l_ij t_ij,k / (2 A_i),         V_k(i,i) = -sum_j V_k(i,j)
  (circulation / area, difference form);
* Laplacian  L(i,j)   = l_ij / (d_ij A_i),             L(i,i)   = -sum_j L(i,j).

Row sums of G, V and L vanish; D is conservative instead.
Dissipation Df = -nu L@L with nu = gamma_h * dxbar^4 / 240,
dxbar = sqrt(4 pi a^2 / N_g).
"""

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .sparse import SparseMatrix

EARTH_RADIUS = 6.37122e6
EARTH_OMEGA = 7.292e-5
GRAVITY = 9.80616
GAMMA_H = 0.04e-2
DT_E = 240.0


def n_cells(level):
    return 10 * 4 ** int(level) + 2


# --------------------------------------------------------------------------
# icosahedron and subdivision
# --------------------------------------------------------------------------

def _icosahedron():
    phi = (1.0 + np.sqrt(5.0)) / 2.0
    v = np.array([
        [-1, phi, 0], [1, phi, 0], [-1, -phi, 0], [1, -phi, 0],
        [0, -1, phi], [0, 1, phi], [0, -1, -phi], [0, 1, -phi],
        [phi, 0, -1], [phi, 0, 1], [-phi, 0, -1], [-phi, 0, 1],
    ], dtype=float)
    v /= np.linalg.norm(v, axis=1)[:, None]
    f = np.array([
        [0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
        [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
        [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
        [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1],
    ], dtype=np.int64)
    return v, _orient_ccw(v, f)


def _orient_ccw(v, f):
    a, b, c = v[f[:, 0]], v[f[:, 1]], v[f[:, 2]]
    flip = np.einsum("ij,ij->i", np.cross(b - a, c - a), a + b + c) < 0
    f = f.copy()
    f[flip, 1], f[flip, 2] = f[flip, 2], f[flip, 1].copy()
    return f


def _bisect(v, f):
    """One level of midpoint bisection, midpoints pushed to the sphere."""
    nv = v.shape[0]
    e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
    lo = np.minimum(e[:, 0], e[:, 1])
    hi = np.maximum(e[:, 0], e[:, 1])
    uniq, inv = np.unique(lo * nv + hi, return_inverse=True)
    ua, ub = uniq // nv, uniq % nv
    mid = v[ua] + v[ub]
    mid /= np.linalg.norm(mid, axis=1)[:, None]
    nf = f.shape[0]
    ab = nv + inv[:nf]
    bc = nv + inv[nf:2 * nf]
    ca = nv + inv[2 * nf:]
    a, b, c = f[:, 0], f[:, 1], f[:, 2]
    nfaces = np.concatenate([
        np.stack([a, ab, ca], 1), np.stack([ab, b, bc], 1),
        np.stack([ca, bc, c], 1), np.stack([ab, bc, ca], 1)])
    return np.concatenate([v, mid]), nfaces


# --------------------------------------------------------------------------
# Hilbert ordering (Skilling's transpose algorithm, vectorised)
# --------------------------------------------------------------------------

def hilbert_keys(points, bits=20):
    """3-D Hilbert index of points in [-1,1]^3 quantised to ``bits`` bits."""
    q = np.clip(((points + 1.0) * 0.5 * ((1 << bits) - 1)).round(), 0,
                (1 << bits) - 1).astype(np.uint64)
    x = [q[:, 0].copy(), q[:, 1].copy(), q[:, 2].copy()]
    one = np.uint64(1)
    m = one << np.uint64(bits - 1)
    qq = m
    while qq > one:
        p = qq - one
        for i in range(3):
            hit = (x[i] & qq) != 0
            t = (x[0] ^ x[i]) & p
            x0_hit = x[0] ^ p
            x0_miss = x[0] ^ t
            xi_miss = x[i] ^ t
            x[0] = np.where(hit, x0_hit, x0_miss)
            if i != 0:
                x[i] = np.where(hit, x[i], xi_miss)
        qq >>= one
    for i in range(1, 3):
        x[i] ^= x[i - 1]
    t = np.zeros_like(x[0])
    qq = m
    while qq > one:
        t = np.where((x[2] & qq) != 0, t ^ (qq - one), t)
        qq >>= one
    for i in range(3):
        x[i] ^= t
    key = np.zeros_like(x[0])
    for b in range(bits - 1, -1, -1):
        bb = np.uint64(b)
        for i in range(3):
            key = (key << one) | ((x[i] >> bb) & one)
    return key


# --------------------------------------------------------------------------
# geometry helpers
# --------------------------------------------------------------------------

def _unit(x):
    return x / np.linalg.norm(x, axis=-1)[..., None]


def _arc(p, q):
    """Great-circle angle between unit vectors (robust atan2 form)."""
    return np.arctan2(np.linalg.norm(np.cross(p, q), axis=-1),
                      np.einsum("...k,...k->...", p, q))


def _sph_tri_area(a, b, c):
    """Area of the unit-sphere triangle abc (Van Oosterom-Strackee)."""
    num = np.abs(np.einsum("...k,...k->...", a, np.cross(b, c)))
    den = (1.0 + np.einsum("...k,...k->...", a, b)
           + np.einsum("...k,...k->...", b, c)
           + np.einsum("...k,...k->...", c, a))
    return 2.0 * np.arctan2(num, den)


@dataclass
class SphereMesh:
    """Voronoi mesh topology/geometry on the unit sphere (Hilbert ordered)."""

    level: int
    x: np.ndarray            # (N,3) cell centres (unit vectors)
    nbr: np.ndarray          # (N,6) neighbours, CCW; pentagons pad with -1
    deg: np.ndarray          # (N,) 5 or 6
    q0: np.ndarray           # (N,6,3) Voronoi edge start (unit vectors)
    q1: np.ndarray           # (N,6,3) Voronoi edge end (CCW about the cell)


def build_mesh(level):
    if level < 0 or level > 11:
        raise ValueError("grid level must lie in 0..11")
    v, f = _icosahedron()
    for _ in range(int(level)):
        v, f = _bisect(v, f)
    nv = v.shape[0]
    # Hilbert renumbering
    order = np.argsort(hilbert_keys(v), kind="stable")
    rank = np.empty(nv, dtype=np.int64)
    rank[order] = np.arange(nv)
    v = v[order]
    f = rank[f]
    cc = _unit(np.cross(v[f[:, 1]] - v[f[:, 0]], v[f[:, 2]] - v[f[:, 0]]))
    # incidences (vertex, face, next-vertex) with the face CCW about vertex
    nf = f.shape[0]
    fid = np.arange(nf)
    inc_v = np.concatenate([f[:, 0], f[:, 1], f[:, 2]])
    inc_p = np.concatenate([f[:, 1], f[:, 2], f[:, 0]])
    inc_f = np.concatenate([fid, fid, fid])
    # angle of the face circumcentre in the vertex tangent frame
    pv = v[inc_v]
    ref = np.where(np.abs(pv[:, 2:3]) < 0.9, np.array([[0.0, 0.0, 1.0]]),
                   np.array([[1.0, 0.0, 0.0]]))
    e1 = _unit(np.cross(ref, pv))
    e2 = np.cross(pv, e1)
    c = cc[inc_f]
    ang = np.arctan2(np.einsum("ij,ij->i", c, e2), np.einsum("ij,ij->i", c, e1))
    srt = np.lexsort((ang, inc_v))
    inc_v, inc_p, inc_f = inc_v[srt], inc_p[srt], inc_f[srt]
    deg = np.bincount(inc_v, minlength=nv)
    if deg.min() < 5 or deg.max() > 6:
        raise RuntimeError("unexpected vertex degree")
    start = np.concatenate([[0], np.cumsum(deg)[:-1]])
    slot = np.arange(inc_v.shape[0]) - start[inc_v]
    nbr = np.full((nv, 6), -1, dtype=np.int64)
    face = np.full((nv, 6), -1, dtype=np.int64)
    nbr[inc_v, slot] = inc_p
    face[inc_v, slot] = inc_f
    # edge k (to nbr k) runs from cc(face k-1) to cc(face k)
    prev_slot = (np.arange(6)[None, :] - 1) % deg[:, None]
    prev_face = np.take_along_axis(face, prev_slot, axis=1)
    valid = nbr >= 0
    q0 = np.zeros((nv, 6, 3))
    q1 = np.zeros((nv, 6, 3))
    q0[valid] = cc[prev_face[valid]]
    q1[valid] = cc[face[valid]]
    return SphereMesh(level=int(level), x=v, nbr=nbr, deg=deg, q0=q0, q1=q1)


@dataclass
class SphereGeometry:
    """Per-(cell, edge) finite-volume quantities, radius included."""

    radius: float
    area: np.ndarray         # (N,) cell areas (m^2)
    length: np.ndarray       # (N,6) Voronoi edge lengths l_ij (m), 0 on pads
    dist: np.ndarray         # (N,6) centre distances d_ij (m), 1 on pads
    normal: np.ndarray       # (N,6,3) outward unit normal at edge midpoint
    tangent: np.ndarray      # (N,6,3) CCW unit tangent at edge midpoint


def mesh_geometry(mesh, radius=EARTH_RADIUS):
    x, nbr = mesh.x, mesh.nbr
    valid = nbr >= 0
    N = x.shape[0]
    xi = np.broadcast_to(x[:, None, :], (N, 6, 3))
    xj = x[np.where(valid, nbr, 0)]
    q0, q1 = mesh.q0, mesh.q1
    length = np.where(valid, radius * _arc(q0, q1), 0.0)
    dist = np.where(valid, radius * _arc(xi, xj), 1.0)
    mid = _unit(np.where(valid[..., None], q0 + q1, xi))
    tang = _unit(np.where(valid[..., None], q1 - q0, np.cross(xi, mid) + 1.0))
    normal = _unit(np.cross(tang, mid))
    tangent = np.cross(mid, normal)
    normal = np.where(valid[..., None], normal, 0.0)
    tangent = np.where(valid[..., None], tangent, 0.0)
    tri = np.where(valid, _sph_tri_area(xi, q0, q1), 0.0)
    area = radius * radius * tri.sum(axis=1)
    return SphereGeometry(radius=radius, area=area, length=length, dist=dist,
                          normal=normal, tangent=tangent)


# --------------------------------------------------------------------------
# operators
# --------------------------------------------------------------------------

@dataclass
class DiscreteOperators:
    """Same fields as expintkit.swe.DiscreteOperators (swe.py:23-46).

    Extra (sphere-only) fields: ``areas`` per cell, ``level`` and the mesh;
    ``cell_area`` is the mean cell area.
    """

    Gx: SparseMatrix
    Gy: SparseMatrix
    Gz: SparseMatrix
    Dx: SparseMatrix
    Dy: SparseMatrix
    Dz: SparseMatrix
    Vx: SparseMatrix
    Vy: SparseMatrix
    Vz: SparseMatrix
    L: SparseMatrix
    Df: SparseMatrix
    n_x: np.ndarray
    n_y: np.ndarray
    n_z: np.ndarray
    f: np.ndarray
    h_s: np.ndarray
    g: float
    nu: float
    n_g: int
    cell_area: float
    areas: np.ndarray = None
    level: int = -1
    mesh: SphereMesh = field(default=None, repr=False)

    def with_surface(self, h_s):
        """Copy sharing every operator, with a new surface height h_s."""
        h_s = np.asarray(h_s, dtype=float)
        if h_s.shape != (self.n_g,):
            raise ValueError("h_s must have one value per cell")
        kw = dict(self.__dict__)
        kw["h_s"] = h_s.copy()
        return DiscreteOperators(**kw)


def dissipation_coefficient(gamma_h, dxbar, dt_e=DT_E, n_gamma=4):
    """nu = gamma_h * dxbar^n_gamma / dt_e (swe.py:65-67)."""
    return gamma_h * dxbar ** n_gamma / dt_e


def _stencil_csr(N, nbr, off, diag):
    """CSR with the diagonal first and the neighbours in CCW slot order,
    then canonicalised (sorted column indices)."""
    valid = nbr >= 0
    cnt = 1 + valid.sum(axis=1)
    indptr = np.concatenate([[0], np.cumsum(cnt)])
    cols = np.concatenate([np.arange(N)[:, None], nbr], axis=1)
    vals = np.concatenate([diag[:, None], off], axis=1)
    keep = np.concatenate([np.ones((N, 1), bool), valid], axis=1)
    m = sp.csr_matrix((vals[keep], cols[keep].astype(np.int32),
                       indptr.astype(np.int32)), shape=(N, N))
    m.sort_indices()
    return m


def _rowsum(a):
    """Sequential (slot-order) row sum, so the order is pinned."""
    s = a[:, 0].copy()
    for k in range(1, a.shape[1]):
        s = s + a[:, k]
    return s


def sphere_operators(level, radius=EARTH_RADIUS, omega=EARTH_OMEGA,
                     g=GRAVITY, gamma_h=GAMMA_H, h_s=None, mesh=None):
    """DiscreteOperators on the icosahedral Voronoi grid of ``level``."""
    mesh = build_mesh(level) if mesh is None else mesh
    geo = mesh_geometry(mesh, radius)
    N = mesh.x.shape[0]
    nbr = mesh.nbr
    two_a = (2.0 * geo.area)[:, None]
    lv = geo.length
    valid = nbr >= 0
    # divergence coefficients l n / (2A)
    dvec = (lv[..., None] * geo.normal) / two_a[..., None]
    # Perot gradient coefficients l a (m - x) / (A d), tangent-projected
    xi = mesh.x[:, None, :]
    mid = _unit(np.where(valid[..., None], mesh.q0 + mesh.q1, xi))
    w = lv / (geo.area[:, None] * geo.dist)
    graw = w[..., None] * (radius * (mid - xi))
    gvec = graw - xi * np.einsum("nk,nsk->ns", mesh.x, graw)[..., None]
    gvec = np.where(valid[..., None], gvec, 0.0)
    vvec = (lv[..., None] * geo.tangent) / two_a[..., None]
    lap = np.where(nbr >= 0, lv / (geo.dist * geo.area[:, None]), 0.0)
    ops = {}
    for k, name in enumerate("xyz"):
        g_off = gvec[..., k]
        d_off = dvec[..., k]
        v_off = vvec[..., k]
        ops["G" + name] = SparseMatrix(_stencil_csr(N, nbr, g_off, -_rowsum(g_off)))
        ops["D" + name] = SparseMatrix(_stencil_csr(N, nbr, d_off, _rowsum(d_off)))
        ops["V" + name] = SparseMatrix(_stencil_csr(N, nbr, v_off, -_rowsum(v_off)))
    Lm = _stencil_csr(N, nbr, lap, -_rowsum(lap))
    dxbar = np.sqrt(4.0 * np.pi * radius * radius / N)
    nu = dissipation_coefficient(gamma_h, dxbar)
    Df = SparseMatrix(-nu * (Lm @ Lm))
    x = mesh.x
    return DiscreteOperators(
        L=SparseMatrix(Lm), Df=Df,
        n_x=x[:, 0].copy(), n_y=x[:, 1].copy(), n_z=x[:, 2].copy(),
        f=2.0 * omega * x[:, 2],
        h_s=np.zeros(N) if h_s is None else np.asarray(h_s, dtype=float),
        g=float(g), nu=float(nu), n_g=int(N),
        cell_area=float(4.0 * np.pi * radius * radius / N),
        areas=geo.area, level=int(level), mesh=mesh, **ops)


_CACHE = {}


def cached_sphere_operators(level):
    """Process-local cache (tests build the same small grids repeatedly)."""
    if level not in _CACHE:
        _CACHE[level] = sphere_operators(level)
    return _CACHE[level]
