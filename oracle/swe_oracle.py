"""Oracle restatement of the shallow-water F(u) and Jacobian.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Works on any object with
the ``DiscreteOperators`` fields of swe.py:23-46 (the sphere grid of
``paper_1805_02144_b200.grid`` or the reference's planar factory).
"""

from types import SimpleNamespace

import numpy as np
import scipy.sparse as sp


def _csr(m):
    return m.csr if hasattr(m, "csr") else m


def _fields(ops, u):
    N = ops.n_g
    u = np.asarray(u, dtype=float)
    if u.shape != (4 * N,):
        raise ValueError(f"state must have length {4 * N}")
    return u[:N], u[N:2 * N], u[2 * N:3 * N], u[3 * N:]


def _eta(ops, ux, uy, uz):
    """swe.py:144-146."""
    return (_csr(ops.Vx) @ ux + _csr(ops.Vy) @ uy + _csr(ops.Vz) @ uz + ops.f)


def _nxu(ops, ux, uy, uz):
    """swe.py:136-141 (n x u, despite the reference comment)."""
    return (ops.n_y * uz - ops.n_z * uy, ops.n_z * ux - ops.n_x * uz,
            ops.n_x * uy - ops.n_y * ux)


def swe_rhs(ops, u):
    """swe.py:149-168."""
    ux, uy, uz, h = _fields(ops, u)
    if not np.all(np.isfinite(u)):
        bad = int(np.flatnonzero(~np.isfinite(u))[0])
        raise ValueError(f"non-finite state entry at index {bad}")
    eta = _eta(ops, ux, uy, uz)
    px, py, pz = _nxu(ops, ux, uy, uz)
    E = 0.5 * (ux * ux + uy * uy + uz * uz) + ops.g * (h + ops.h_s)
    Df = _csr(ops.Df)
    fx = -eta * px - _csr(ops.Gx) @ E + Df @ ux
    fy = -eta * py - _csr(ops.Gy) @ E + Df @ uy
    fz = -eta * pz - _csr(ops.Gz) @ E + Df @ uz
    fh = -(_csr(ops.Dx) @ (ux * h) + _csr(ops.Dy) @ (uy * h)
           + _csr(ops.Dz) @ (uz * h)) + Df @ h
    return np.concatenate([fx, fy, fz, fh])


def swe_jacobian(ops, u):
    """swe.py:175-223: J = (J_v + J_r) + J_m as a 4N x 4N scipy CSR; its
    ``nnz`` (scipy's zero-dropping rules) is the engine's n_A."""
    ux, uy, uz, h = _fields(ops, u)
    eta = _eta(ops, ux, uy, uz)
    px, py, pz = _nxu(ops, ux, uy, uz)
    N = ops.n_g
    Z = sp.csr_matrix((N, N))
    d = lambda a: sp.diags(a, format="csr")  # noqa: E731
    Vx, Vy, Vz = _csr(ops.Vx), _csr(ops.Vy), _csr(ops.Vz)
    Gx, Gy, Gz = _csr(ops.Gx), _csr(ops.Gy), _csr(ops.Gz)
    Dx, Dy, Dz = _csr(ops.Dx), _csr(ops.Dy), _csr(ops.Dz)
    Df = _csr(ops.Df)
    Jv = -sp.bmat([[d(px) @ Vx, d(px) @ Vy, d(px) @ Vz, Z],
                   [d(py) @ Vx, d(py) @ Vy, d(py) @ Vz, Z],
                   [d(pz) @ Vx, d(pz) @ Vy, d(pz) @ Vz, Z],
                   [Z, Z, Z, Z]], format="csr")
    ex, ey, ez = d(eta * ops.n_x), d(eta * ops.n_y), d(eta * ops.n_z)
    Jr = sp.bmat([[Df, ez, -ey, Z], [-ez, Df, ex, Z], [ey, -ex, Df, Z],
                  [Z, Z, Z, Df]], format="csr")
    Jm = -sp.bmat([[Gx @ d(ux), Gx @ d(uy), Gx @ d(uz), ops.g * Gx],
                   [Gy @ d(ux), Gy @ d(uy), Gy @ d(uz), ops.g * Gy],
                   [Gz @ d(ux), Gz @ d(uy), Gz @ d(uz), ops.g * Gz],
                   [Dx @ d(h), Dy @ d(h), Dz @ d(h),
                    Dx @ d(ux) + Dy @ d(uy) + Dz @ d(uz)]], format="csr")
    J = Jv + Jr + Jm
    return SimpleNamespace(csr=J, matvec=J.dot, n_rows=J.shape[0], nnz=J.nnz)


def swe_jv_matrix_free(ops, u, v):
    """J v without assembling J (Df applied as
    -nu L(L .)).  Used to cross-check the assembled oracle."""
    ux, uy, uz, h = _fields(ops, u)
    ax, ay, az, b = _fields(ops, v)
    eta = _eta(ops, ux, uy, uz)
    px, py, pz = _nxu(ops, ux, uy, uz)
    L = _csr(ops.L)
    zeta = _csr(ops.Vx) @ ax + _csr(ops.Vy) @ ay + _csr(ops.Vz) @ az
    e = ux * ax + uy * ay + uz * az + ops.g * b
    cx, cy, cz = _nxu(ops, ax, ay, az)

    def df(q):
        return -ops.nu * (L @ (L @ q))

    jx = -px * zeta - eta * cx - _csr(ops.Gx) @ e + df(ax)
    jy = -py * zeta - eta * cy - _csr(ops.Gy) @ e + df(ay)
    jz = -pz * zeta - eta * cz - _csr(ops.Gz) @ e + df(az)
    jh = -(_csr(ops.Dx) @ (h * ax + ux * b) + _csr(ops.Dy) @ (h * ay + uy * b)
           + _csr(ops.Dz) @ (h * az + uz * b)) + df(b)
    return np.concatenate([jx, jy, jz, jh])


def swe_problem(ops):
    """SemilinearProblem-like closure pair (harness.py:184-189)."""
    return SimpleNamespace(n=4 * ops.n_g, f=lambda u: swe_rhs(ops, u),
                           jac=lambda u: swe_jacobian(ops, u))
