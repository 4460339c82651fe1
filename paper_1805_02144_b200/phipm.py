"""GPU ``phipm_simul_iom2`` behind the reference's engine API.

Mirrors /root/reference/pkg/src/expintkit/phipm.py: ``PhiTask`` (87-125),
``PhipmResult`` (140-156), ``PhipmFailure`` (34-42), ``MatvecOperator``
(45-54), ``as_operator`` (73-84), ``cost_estimate`` (217-238) and
``phipm_simul_iom2`` (291-370).  The whole engine call -- w recurrence,
IOM2 Krylov sweep, augmented-matrix exponential, (tau, m) controller -- runs
as one cooperative kernel on the GPU (``eik_csr_phipm`` / ``eik_swe_phipm``);
this module only validates the task and moves vectors across the C ABI.

Operators the device engine accepts: ``SparseMatrix`` / scipy sparse /
dense ``ndarray`` (a device CSR operator), a ``DeviceOperator`` such as
``swe.assemble_jacobian(ops, u)`` or ``scaled(op, dt)``, or a
``MatvecOperator``.  A ``MatvecOperator`` around an arbitrary Python callable
keeps the engine on the device and calls back to the host for every matvec
(``eik_cb_phipm``: a mailbox in mapped memory, one PCIe round trip per
product); everything else about the call is identical.
"""

import csv
import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse

from . import _native as nat
from .sparse import SparseMatrix

MAX_SUBSTEPS = 10 ** 6
DENSE_SIZE_CAP = 256        # kernels.py:20
CRAWL_SUBSTEPS = 100
PADE13_THETA = 5.37


class PhipmFailure(RuntimeError):
    """Engine failed to converge within the substep budget (phipm.py:34)."""

    def __init__(self, message, *, t_reached, substeps, rejections, matvecs):
        super().__init__(message)
        self.t_reached = t_reached
        self.substeps = substeps
        self.rejections = rejections
        self.matvecs = matvecs


class DeviceOperator:
    """An operator the device engine can apply: ``kind`` is "csr" or "swe"."""

    kind = None
    n = 0
    nnz = 0
    scale = 1.0

    def scaled(self, alpha):
        raise NotImplementedError


class CsrDeviceOperator(DeviceOperator):
    """A x = scale * (M x) for a host CSR matrix M, applied on the device."""

    kind = "csr"

    def __init__(self, csr, scale=1.0, nnz=None):
        self.csr = scipy.sparse.csr_matrix(csr, dtype=float)
        if self.csr.shape[0] != self.csr.shape[1]:
            raise ValueError("operator must be square")
        self.n = self.csr.shape[0]
        self.nnz = int(self.csr.nnz if nnz is None else nnz)
        self.scale = float(scale)

    def scaled(self, alpha):
        return CsrDeviceOperator(self.csr, self.scale * float(alpha), self.nnz)


class MatvecOperator:
    """Abstract operator: a matvec plus n, nnz (phipm.py:45-54)."""

    def __init__(self, matvec, n, nnz):
        self._matvec = matvec
        self.n = n
        self.nnz = nnz

    def matvec(self, x):
        return self._matvec(x)


def as_operator(A, n=None):
    """phipm.py:73-84, returning a device operator where possible."""
    if isinstance(A, (DeviceOperator, MatvecOperator)):
        return A
    if isinstance(A, SparseMatrix) or hasattr(A, "csr"):
        return CsrDeviceOperator(A.csr)
    if scipy.sparse.issparse(A):
        return CsrDeviceOperator(A.tocsr())
    if isinstance(A, np.ndarray):
        A = np.asarray(A, dtype=float)
        return CsrDeviceOperator(scipy.sparse.csr_matrix(A),
                                 nnz=int(np.count_nonzero(A)))
    raise TypeError(f"cannot interpret {type(A)!r} as an operator")


class HostMatvecOperator(DeviceOperator):
    """A ``MatvecOperator`` around an arbitrary host callable: the engine runs
    on the device and requests every matvec from the host through a mailbox
    in mapped memory (``eik_cb_phipm``): one PCIe round trip plus the
    callable per performed product -- slow, as the plug point allows."""

    kind = "host"

    def __init__(self, op, scale=1.0):
        self.op = op
        self.n = int(op.n)
        self.nnz = int(op.nnz)
        self.scale = float(scale)

    def scaled(self, alpha):
        return HostMatvecOperator(self.op, self.scale * float(alpha))


def _device_operator(op):
    if isinstance(op, DeviceOperator):
        return op
    if isinstance(op, MatvecOperator):
        dev = getattr(op, "device", None) or getattr(op._matvec, "device", None)
        if isinstance(dev, DeviceOperator):
            return dev
        return HostMatvecOperator(op)
    return as_operator(op)


_CB_CACHE = {}


def _cb_context(n, m_cap):
    key = (n, m_cap)
    ctx = _CB_CACHE.get(key)
    if ctx is None:
        h = nat.C.c_void_p()
        nat.check(nat.load().eik_cb_create(n, 0, int(m_cap), nat.C.byref(h)), "eik_cb_create")
        ctx = _CbCtx(h)
        if len(_CB_CACHE) > 4:
            _CB_CACHE.clear()
        _CB_CACHE[key] = ctx
    return ctx


class _CbCtx:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            nat.load().eik_cb_destroy(self.h)
        except Exception:
            pass


def _run_host_callback(op, t, W, info, trace, cap, tlen):
    """eik_cb_phipm with op.op.matvec as the callback; an exception raised by
    the callable aborts the device engine and is re-raised here."""
    n = op.n
    failure = []

    def cb(_user, xp, yp, nn):
        try:
            x = np.ctypeslib.as_array(xp, shape=(nn,)).copy()
            y = np.asarray(op.op.matvec(x), dtype=float)
            if y.shape != (nn,):
                raise ValueError(f"matvec returned shape {y.shape}, expected ({nn},)")
            np.ctypeslib.as_array(yp, shape=(nn,))[:] = y
            return 0
        except BaseException as e:  # noqa: BLE001 -- re-raised after the call
            failure.append(e)
            return 1

    fn = nat.MATVEC_FN(cb)
    ctx = _cb_context(n, min(max(t.m_max, 1), n, DENSE_SIZE_CAP))
    st = nat.load().eik_cb_phipm(ctx.h, fn, None, op.scale, op.nnz, nat.C.byref(t),
                                 nat.dptr(W), nat.C.byref(info), trace, cap,
                                 nat.C.byref(tlen))
    if failure:
        raise failure[0]
    return st


@dataclass
class PhiTask:
    """One engine request (phipm.py:87-125), same fields and validation."""

    A: object
    v: list
    rho: list
    tol: float = 1e-4
    m_init: int = 1
    iom: int = 2
    m_max: int = 100
    delta: float = 1.4
    tau_init: float | None = None
    zero_skip: bool = True
    trace: bool = False

    def __post_init__(self):
        self.v = [np.asarray(vl, dtype=float) for vl in self.v]
        if not self.v:
            raise ValueError("at least one input vector is required")
        n = self.v[0].shape[0]
        if any(vl.shape != (n,) for vl in self.v):
            raise ValueError("all input vectors must have the same length")
        if not any(vl.any() for vl in self.v):
            raise ValueError("at least one input vector must be nonzero")
        rho = [float(r) for r in self.rho]
        if not rho or rho[0] <= 0.0 or rho[-1] > 1.0:
            raise ValueError("rho must lie in (0, 1]")
        if any(b <= a for a, b in zip(rho, rho[1:])):
            raise ValueError("rho must be strictly ascending")
        self.rho = rho
        if self.tol <= 0.0:
            raise ValueError("tol must be positive")


@dataclass
class PhipmResult:
    W: np.ndarray
    substeps: int
    rejections: int
    matvecs: int
    tau_final: float
    m_final: int
    trace: list = field(default_factory=list)

    def write_trace_csv(self, path):
        """Serialize the per-substep trace (phipm.py:150-156)."""
        with open(path, "w", newline="") as fh:
            writer = csv.writer(fh)
            writer.writerow(["attempt", "t", "tau", "m", "eps_m", "omega",
                             "accepted"])
            writer.writerows(self.trace)


def cost_estimate(tau, m, N, n_A, p, norm_hhat, t_out, t_k):
    """phipm.py:217-238 (host copy of the device controller's cost model;
    the device evaluates csrc/eik_control.h::cost_estimate)."""
    if tau <= 0.0:
        raise ValueError("tau must be positive")
    M = 44.0 / 3.0
    if norm_hhat > PADE13_THETA:
        M += 2.0 * math.ceil(math.log2(norm_hhat / PADE13_THETA))
    substeps = math.ceil((t_out - t_k) / tau) if t_out > t_k else 1
    return substeps * (m * (N + n_A) + 2 * max(p - 1, 0) * (n_A + N)
                       + M * (m + p + 1) ** 3 + (2 * p + 1) * N)


_CSR_CACHE = {}


def _csr_context(op, m_cap):
    key = (id(op.csr), op.n, op.nnz, m_cap)
    ent = _CSR_CACHE.get(key)
    if ent is not None and ent[0] is op.csr:
        return ent[1]
    lib = nat.load()
    view, keep = nat.csr_view(op.csr)
    h = nat.C.c_void_p()
    nat.check(lib.eik_csr_create(op.n, view, 0, int(m_cap), nat.C.byref(h)),
              "eik_csr_create")
    ctx = _CsrCtx(h)
    if len(_CSR_CACHE) > 8:
        _CSR_CACHE.clear()
    _CSR_CACHE[key] = (op.csr, ctx)
    return ctx


class _CsrCtx:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            nat.load().eik_csr_destroy(self.h)
        except Exception:
            pass


def _run(task, op):
    lib = nat.load()
    n = task.v[0].shape[0]
    if op.n != n:
        raise ValueError("operator and vector sizes differ")
    ns = len(task.rho)
    t, keep = nat.make_task(task.v, task.rho, task.tol, task.m_init, task.iom,
                            task.m_max, task.delta, task.tau_init,
                            task.zero_skip, MAX_SUBSTEPS)
    cap = 4096 if task.trace else 0
    while True:
        info = nat.EikPhipmInfo()
        trace = (nat.EikTraceRec * max(cap, 1))()
        tlen = nat.C.c_int64(0)
        W = np.zeros((ns, n))
        if op.kind == "csr":
            ctx = _csr_context(op, min(max(task.m_max, 1), n, DENSE_SIZE_CAP))
            st = lib.eik_csr_phipm(ctx.h, op.scale, int(op.nnz), nat.C.byref(t),
                                   nat.dptr(W), nat.C.byref(info),
                                   trace if cap else None, cap, nat.C.byref(tlen))
        elif op.kind == "swe":
            st = op.run_phipm(t, W, info, trace if cap else None, cap, tlen)
        elif op.kind == "host":
            st = _run_host_callback(op, t, W, info, trace if cap else None, cap, tlen)
        else:
            raise TypeError(f"unsupported device operator {op!r}")
        # the trace is unbounded (phipm.py:341-343): the device counts every
        # attempt; a call with more attempts than the buffer holds is re-run
        # (deterministically) with a buffer of the right size
        if cap and st == nat.EIK_OK and tlen.value > cap:
            cap = int(tlen.value)
            continue
        break
    if st == nat.EIK_EPHIPM:
        raise PhipmFailure(
            f"no convergence within {MAX_SUBSTEPS} substeps "
            f"(t reached {info.t_reached:.3e})",
            t_reached=info.t_reached, substeps=info.substeps,
            rejections=info.rejections, matvecs=info.matvecs)
    nat.check(st, "phipm_simul_iom2")
    rows = []
    for k in range(min(tlen.value, cap)):
        r = trace[k]
        rows.append((int(r.attempt), r.t, r.tau, int(r.m), r.eps_m, r.omega,
                     bool(r.accepted)))
    return PhipmResult(W=np.ascontiguousarray(W.T), substeps=int(info.substeps),
                       rejections=int(info.rejections),
                       matvecs=int(info.matvecs), tau_final=float(info.tau_final),
                       m_final=int(info.m_final), trace=rows)


def phipm_simul_iom2(task):
    """Evaluate all requested phi linear combinations in one sweep (GPU).

    W[:, i] = sum_l rho_i^l phi_l(rho_i A) v_l with every rho_i landed on
    exactly; raises PhipmFailure when the substep budget is exhausted.
    """
    return _run(task, _device_operator(task.A))
