"""Shallow-water F(u), J(u) v and nnz(J) on the GPU, reference API.

Mirrors /root/reference/pkg/src/expintkit/swe.py: ``DiscreteOperators``
(23-46), ``split_state``/``stack_state`` (124-133), ``rhs`` (149-168),
``assemble_jacobian`` (220-223; here a device operator: matrix-free J v plus
the exact scipy nnz), ``dissipation_coefficient`` (65-67).  One ``SweContext``
(C-ABI ``EikSwe``) is created per operator set and cached; it owns the
device copy of the grid (ELL stencil built from the CSR operators), the
resident trajectory state and the engine's warm-start seeds.
"""

import ctypes as C
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .grid import DiscreteOperators, dissipation_coefficient  # noqa: F401
from .phipm import DeviceOperator, MatvecOperator

_OP_ORDER = ("Gx", "Gy", "Gz", "Dx", "Dy", "Dz", "Vx", "Vy", "Vz", "L", "Df")


def _periodic_diff(n, dx):
    """Centred periodic first derivative (swe.py:70-76)."""
    import scipy.sparse as sp
    e = np.ones(n) / (2.0 * dx)
    D = sp.diags([e[:-1], -e[:-1]], [1, -1], shape=(n, n), format="lil")
    D[0, n - 1] = -1.0 / (2.0 * dx)
    D[n - 1, 0] = 1.0 / (2.0 * dx)
    return sp.csr_matrix(D)


def _periodic_second(n, dx):
    """Periodic second derivative (swe.py:79-86)."""
    import scipy.sparse as sp
    e = np.ones(n) / dx ** 2
    D = sp.diags([e[:-1], -2.0 * e, e[:-1]], [1, 0, -1], shape=(n, n), format="lil")
    D[0, n - 1] = 1.0 / dx ** 2
    D[n - 1, 0] = 1.0 / dx ** 2
    return sp.csr_matrix(D)


def planar_periodic_operators(nx, ny, dx, f0=1e-4, g=9.80616, gamma_h=0.04e-2, h_s=None):
    """The reference's doubly periodic planar operator set (swe.py:89-121):
    centred differences, n = z-hat, Vx = -d/dy, Vy = d/dx, Df = -nu L@L.
    Nodes row-major, index = iy * nx + ix."""
    import scipy.sparse as sp
    from .sparse import SparseMatrix
    if nx < 4 or ny < 4:
        raise ValueError("grid must be at least 4x4")
    if dx <= 0.0:
        raise ValueError("dx must be positive")
    n_g = nx * ny
    Ix = sp.identity(nx, format="csr")
    Iy = sp.identity(ny, format="csr")
    ddx = sp.kron(Iy, _periodic_diff(nx, dx), format="csr")
    ddy = sp.kron(_periodic_diff(ny, dx), Ix, format="csr")
    lap = (sp.kron(Iy, _periodic_second(nx, dx)) + sp.kron(_periodic_second(ny, dx), Ix)).tocsr()
    zero = sp.csr_matrix((n_g, n_g))
    nu = dissipation_coefficient(gamma_h, dx)
    return DiscreteOperators(
        Gx=SparseMatrix(ddx), Gy=SparseMatrix(ddy), Gz=SparseMatrix(zero),
        Dx=SparseMatrix(ddx), Dy=SparseMatrix(ddy), Dz=SparseMatrix(zero),
        Vx=SparseMatrix(-ddy), Vy=SparseMatrix(ddx), Vz=SparseMatrix(zero),
        L=SparseMatrix(lap), Df=SparseMatrix(-nu * (lap @ lap)),
        n_x=np.zeros(n_g), n_y=np.zeros(n_g), n_z=np.ones(n_g), f=np.full(n_g, float(f0)),
        h_s=np.zeros(n_g) if h_s is None else np.asarray(h_s, dtype=float),
        g=float(g), nu=nu, n_g=n_g, cell_area=dx * dx)


def gaussian_hill_state(ops, nx, ny, dx, h0=8000.0, amplitude=100.0, sigma_cells=None,
                        center=None):
    """Rest state with a Gaussian bump in the height field (swe.py:240-253)."""
    if sigma_cells is None:
        sigma_cells = nx / 8.0
    if center is None:
        center = (nx / 2.0, ny / 2.0)
    X, Y = np.meshgrid(np.arange(nx), np.arange(ny))
    r2 = (X - center[0]) ** 2 + (Y - center[1]) ** 2
    h = h0 + amplitude * np.exp(-r2 / (2.0 * sigma_cells ** 2))
    z = np.zeros(ops.n_g)
    return stack_state(z, z.copy(), z.copy(), h.ravel())


def split_state(ops, state):
    n = ops.n_g
    state = np.asarray(state, dtype=float)
    if state.shape != (4 * n,):
        raise ValueError(f"state must have length {4 * n}")
    return state[:n], state[n:2 * n], state[2 * n:3 * n], state[3 * n:]


def stack_state(ux, uy, uz, h):
    return np.concatenate([ux, uy, uz, h])


class SweContext:
    """Device context for one operator set (owns an ``EikSwe``)."""

    def __init__(self, ops, device=0, m_max=100):
        lib = nat.load()
        self.ops = ops
        self.n_g = int(ops.n_g)
        self.n = 4 * self.n_g
        views = (nat.EikCsrView * 11)()
        keep = []
        for k, name in enumerate(_OP_ORDER):
            v, kp = nat.csr_view(getattr(ops, name))
            views[k] = v
            keep.append(kp)
        fields = [np.ascontiguousarray(getattr(ops, f), dtype=float)
                  for f in ("n_x", "n_y", "n_z", "f", "h_s")]
        h = C.c_void_p()
        st = lib.eik_swe_create(self.n_g, views, *(nat.dptr(a) for a in fields),
                                float(ops.g), float(ops.nu), int(device),
                                int(m_max), C.byref(h))
        nat.check(st, "eik_swe_create")
        self.h = h
        self._fin = weakref.finalize(self, lib.eik_swe_destroy, h)

    # --------------------------------------------------------------- basics
    def _vec(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ValueError(f"state must have length {self.n}")
        return x

    def rhs(self, u):
        u = self._vec(u)
        out = np.empty(self.n)
        nat.check(nat.load().eik_swe_rhs(self.h, nat.dptr(u), nat.dptr(out)),
                  "rhs")
        return out

    def jv(self, u, v):
        u, v = self._vec(u), self._vec(v)
        out = np.empty(self.n)
        nat.check(nat.load().eik_swe_jv(self.h, nat.dptr(u), nat.dptr(v),
                                        nat.dptr(out)), "J v")
        return out

    def jac_nnz(self, u):
        u = self._vec(u)
        r = C.c_int64(0)
        nat.check(nat.load().eik_swe_jac_nnz(self.h, nat.dptr(u), C.byref(r)),
                  "nnz(J)")
        return int(r.value)

    def set_state(self, u):
        u = self._vec(u)
        nat.check(nat.load().eik_swe_set_state(self.h, nat.dptr(u)), "set_state")

    def get_state(self):
        out = np.empty(self.n)
        nat.check(nat.load().eik_swe_get_state(self.h, nat.dptr(out)),
                  "get_state")
        return out

    def set_prev(self, u_prev):
        if u_prev is None:
            nat.check(nat.load().eik_swe_set_prev(self.h, None), "set_prev")
            return
        u = self._vec(u_prev)
        nat.check(nat.load().eik_swe_set_prev(self.h, nat.dptr(u)), "set_prev")

    def step(self, scheme, dt, tol):
        """One resident-state step; returns the per-engine-call infos."""
        calls = (nat.EikPhipmInfo * 3)()
        nc = C.c_int32(0)
        st = nat.load().eik_swe_step(self.h, nat.SCHEME_IDS[scheme], float(dt),
                                     float(tol), calls, C.byref(nc))
        if st == nat.EIK_EPHIPM:
            from .phipm import PhipmFailure
            bad = [c for c in calls[:nc.value] if c.status == nat.EIK_EPHIPM]
            c = bad[0] if bad else calls[0]
            raise PhipmFailure("no convergence within the substep budget",
                               t_reached=c.t_reached, substeps=c.substeps,
                               rejections=c.rejections, matvecs=c.matvecs)
        nat.check(st, f"step {scheme}")
        return [calls[k] for k in range(nc.value)]

    def seeds(self, slot):
        tau = C.c_double(0.0)
        m = C.c_int64(0)
        nat.check(nat.load().eik_swe_seeds(self.h, nat.SLOT_IDS[slot],
                                           C.byref(tau), C.byref(m), 0), "seeds")
        return (tau.value if tau.value > 0 else None), int(m.value)

    def set_seeds(self, slot, tau, m):
        t = C.c_double(tau if tau else -1.0)
        mm = C.c_int64(int(m))
        nat.check(nat.load().eik_swe_seeds(self.h, nat.SLOT_IDS[slot],
                                           C.byref(t), C.byref(mm), 1), "seeds")

    def reset_seeds(self):
        nat.check(nat.load().eik_swe_reset_seeds(self.h), "reset_seeds")

    def snapshot(self, restore=False):
        """Device-side save (or restore) of state, epi3 history and seeds."""
        nat.check(nat.load().eik_swe_snapshot(self.h, 1 if restore else 0), "snapshot")

    def launches(self):
        return int(nat.load().eik_swe_launches(self.h))

    def krylov_iters(self):
        return int(nat.load().eik_swe_krylov_iters(self.h))

    def last_kernel_ms(self):
        return float(nat.load().eik_swe_last_kernel_ms(self.h))

    def set_hostloop(self, on=True):
        """Launch the split step kernel by kernel (no CUDA graph): every
        Krylov sweep is timed with CUDA events and ncu can profile it."""
        nat.check(nat.load().eik_swe_set_hostloop(self.h, 1 if on else 0), "set_hostloop")

    def sweep_timing(self, reset=False):
        """(ms, sweeps) of the Krylov sweep kernels run in host-loop mode."""
        ms = C.c_double(0.0)
        n = C.c_int64(0)
        nat.check(nat.load().eik_swe_sweep_timing(self.h, C.byref(ms), C.byref(n),
                                                  1 if reset else 0), "sweep_timing")
        return float(ms.value), int(n.value)


_CTX = {}


def context(ops):
    """The cached SweContext of an operator set."""
    key = id(ops)
    ent = _CTX.get(key)
    if ent is not None and ent[0]() is ops:
        return ent[1]
    ctx = SweContext(ops)
    def _drop(_r, k=key, table=_CTX):
        if table is not None:
            table.pop(k, None)

    try:
        ref = weakref.ref(ops, _drop)
    except TypeError:
        ref = (lambda o: (lambda: o))(ops)
    _CTX[key] = (ref, ctx)
    return ctx


def rhs(ops, state):
    """Tendency of [u_x; u_y; u_z; h] (swe.py:149-168), computed on the GPU.
    Raises ValueError on a non-finite state or tendency."""
    return context(ops).rhs(state)


@dataclass
class Diagnostics:
    """Weighted conserved totals and drifts relative to t=0 (swe.py:49-62)."""

    mass: float
    energy: float
    enstrophy: float

    def drifts(self, initial):
        return ((self.mass - initial.mass) / initial.mass,
                (self.energy - initial.energy) / initial.energy,
                (self.enstrophy - initial.enstrophy) / initial.enstrophy)


def diagnostics(ops, state=None, area_weighted=False):
    """Totals of mass (h), energy (g h + |u|^2/2) and potential enstrophy
    ((zeta+f)^2 / 2h) on the GPU (swe.py:226-237).  The reference weights
    every cell by the scalar ``ops.cell_area``; ``area_weighted=True`` uses
    the sphere grid's per-cell areas.  ``state=None`` reads the context's
    resident trajectory state without a host copy."""
    ctx = context(ops)
    out = np.zeros(3)
    u = None if state is None else ctx._vec(state)
    w = np.ascontiguousarray(ops.areas, dtype=float) if area_weighted else None
    nat.check(nat.load().eik_swe_diagnostics(
        ctx.h, None if u is None else nat.dptr(u), None if w is None else nat.dptr(w),
        float(ops.cell_area), nat.dptr(out)), "diagnostics")
    return Diagnostics(mass=float(out[0]), energy=float(out[1]), enstrophy=float(out[2]))


class SweJacobian(DeviceOperator):
    """J(u) (swe.py:175-223) as a device operator: ``matvec`` runs the
    matrix-free stencil J v on the GPU and ``nnz`` is the exact nnz the
    reference's assembled scipy CSR would have (the engine's n_A)."""

    kind = "swe"

    def __init__(self, ops, state, scale=1.0, _nnz=None):
        self.ctx = context(ops)
        self.state = np.ascontiguousarray(state, dtype=float).copy()
        if not np.all(np.isfinite(self.state)):
            raise ValueError("state must be finite")
        self.n = self.ctx.n
        self.n_rows = self.n
        self.scale = float(scale)
        self._nnz = _nnz

    @property
    def nnz(self):
        if self._nnz is None:
            self._nnz = self.ctx.jac_nnz(self.state)
        return self._nnz

    def matvec(self, x):
        out = self.ctx.jv(self.state, x)
        return out if self.scale == 1.0 else self.scale * out

    def scaled(self, alpha):
        return SweJacobian(self.ctx.ops, self.state, self.scale * float(alpha),
                           self._nnz)

    def as_matvec_operator(self):
        op = MatvecOperator(self.matvec, self.n, self.nnz)
        op.device = self
        return op

    def run_phipm(self, task, W, info, trace, cap, tlen):
        u = self.state
        return nat.load().eik_swe_phipm(
            self.ctx.h, nat.dptr(u), self.scale, C.byref(task), nat.dptr(W),
            C.byref(info), trace, cap, C.byref(tlen))


def assemble_jacobian(ops, state):
    """Full 4N x 4N tendency Jacobian as a device operator."""
    return SweJacobian(ops, state)


def jacobian_nnz(ops, state):
    return context(ops).jac_nnz(state)
