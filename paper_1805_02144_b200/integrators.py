"""Exponential Rosenbrock / multistep steps on the GPU, reference API.

Mirrors /root/reference/pkg/src/expintkit/integrators.py: ``SCHEME_NAMES``
(20), ``SemilinearProblem`` (23-61), ``StepRecord`` (64-70), ``EngineSeeds``
(73-83), ``linearize`` (86-104), ``step_rb_euler`` / ``step_epi3`` /
``step_exprb42`` / ``step_pexprb43`` / ``step_exprb53`` (140-224) and
``integrate`` (318-369).

Two execution routes, both with every engine call on the device:

* shallow-water problems (``swe_problem(ops)``): the whole step -- F(u_n),
  eta, n_A, the 2-3 engine calls, the stage perturbations D(U) and the
  stage combinations -- is one cooperative kernel (``eik_swe_step``,
  replayed from a CUDA graph); the state stays resident between steps.
* any other ``SemilinearProblem``: F and J are the user's host callables,
  so the step logic runs here and each engine call is a device call with
  A = dt * J(u_n) as a device CSR operator (integrators.py:115-117).
"""

from dataclasses import dataclass

import numpy as np

from . import swe as _swe
from .phipm import (CsrDeviceOperator, HostMatvecOperator, MatvecOperator, PhiTask,
                    phipm_simul_iom2)
from .sparse import SparseMatrix

SCHEME_NAMES = ("rb_euler", "epi3", "exprb42", "pexprb43", "exprb53")


@dataclass
class SemilinearProblem:
    """Stiff ODE u' = F(u) with an analytic Jacobian (integrators.py:23)."""

    n: int
    f: callable
    jac: callable = None
    exact: callable = None
    name: str = ""
    ops: object = None          # set for shallow-water problems

    def rhs(self, u):
        out = np.asarray(self.f(u), dtype=float)
        if not np.all(np.isfinite(out)):
            raise ValueError("non-finite right-hand side")
        return out

    def jacobian(self, u):
        if self.jac is None:
            raise ValueError("the device engine needs an analytic Jacobian")
        return self.jac(u)


def swe_problem(ops):
    """Shallow-water problem on an operator set (harness.py:184-189)."""
    return SemilinearProblem(n=4 * ops.n_g, f=lambda u: _swe.rhs(ops, u),
                             jac=lambda u: _swe.assemble_jacobian(ops, u),
                             name="swe", ops=ops)


@dataclass
class StepRecord:
    t: float
    u: np.ndarray
    dt: float
    matvecs: int = 0
    substeps: int = 0


class EngineSeeds:
    """Warm-start store: final (tau, m) per engine-call slot."""

    def __init__(self):
        self._seeds = {}

    def get(self, slot):
        return self._seeds.get(slot, (None, 1))

    def put(self, slot, result):
        self._seeds[slot] = (result.tau_final, result.m_final)

    def set(self, slot, tau, m):
        self._seeds[slot] = (tau, m)


class _StepStats:
    __slots__ = ("matvecs", "substeps")

    def __init__(self):
        self.matvecs = 0
        self.substeps = 0


_SLOTS = {"rb_euler": ("rbe",), "epi3": ("epi3",),
          "exprb42": ("exprb42/1", "exprb42/2"),
          "pexprb43": ("pexprb43/1", "pexprb43/2"),
          "exprb53": ("exprb53/1", "exprb53/2", "exprb53/3")}


# ------------------------------------------------------------ device route

def _swe_step(problem, scheme, u_n, dt, tol, seeds, stats, u_prev=None):
    if dt <= 0.0:
        raise ValueError("dt must be positive")
    ctx = _swe.context(problem.ops)
    u_n = np.asarray(u_n, dtype=float)
    if scheme not in ("rb_euler", "epi3") and not np.all(np.isfinite(u_n)):
        raise ValueError("state must be finite")
    ctx.set_state(u_n)
    if scheme == "epi3":
        if u_prev is None:
            raise ValueError("epi3 requires the previous state")
        ctx.set_prev(u_prev)
    slots = _SLOTS[scheme]
    # seeds=None starts every engine call cold, (tau, m) = (None, 1)
    # (integrators.py:128); the context's device seeds from an earlier call
    # must not leak into this one.
    for s in slots:
        ctx.set_seeds(s, *(seeds.get(s) if seeds is not None else (None, 1)))
    calls = ctx.step(scheme, dt, tol)
    if seeds is not None:
        for s, c in zip(slots, calls):
            if not c.skipped:
                seeds.set(s, c.tau_final, int(c.m_final))
    if stats is not None:
        for c in calls:
            stats.matvecs += int(c.matvecs)
            stats.substeps += int(c.substeps)
    return ctx.get_state()


# -------------------------------------------------------------- host route

def _device_jacobian(problem, u):
    J = problem.jacobian(u)
    if isinstance(J, _swe.SweJacobian):
        return J
    if isinstance(J, MatvecOperator):
        return HostMatvecOperator(J)
    if not isinstance(J, SparseMatrix):
        J = SparseMatrix(J)
    return CsrDeviceOperator(J.csr)


def linearize(problem, u_n):
    """(J_n, N_n, D, F_n) (integrators.py:86-104); J_n is a device
    operator whose ``matvec`` runs on the GPU."""
    u_n = np.asarray(u_n, dtype=float)
    if not np.all(np.isfinite(u_n)):
        raise ValueError("state must be finite")
    J = problem.jacobian(u_n)
    f_n = problem.rhs(u_n)

    def remainder(u):
        return problem.rhs(u) - J.matvec(u)

    def perturbation(U):
        return problem.rhs(U) - f_n - J.matvec(U - u_n)

    return J, remainder, perturbation, f_n


def _engine(A, vectors, rho, tol, seeds, slot, stats):
    """integrators.py:120-137 with A a device operator (scaled by dt)."""
    p = max(vectors)
    n = next(iter(vectors.values())).shape[0]
    v = [vectors.get(k, np.zeros(n)) for k in range(p + 1)]
    if not any(vl.any() for vl in v):
        return np.zeros((n, len(rho)))
    tau0, m0 = seeds.get(slot) if seeds is not None else (None, 1)
    res = phipm_simul_iom2(PhiTask(A=A, v=v, rho=list(rho), tol=tol,
                                   m_init=m0, tau_init=tau0))
    if seeds is not None:
        seeds.put(slot, res)
    if stats is not None:
        stats.matvecs += res.matvecs
        stats.substeps += res.substeps
    return res.W


def _matvec(J, x):
    if isinstance(J, CsrDeviceOperator):
        return J.csr @ x  # host-side stage algebra on the user's own matrix
    if isinstance(J, HostMatvecOperator):
        return J.op.matvec(x)  # the user's own host callable
    return J.matvec(x)


def _host_step(problem, scheme, u, dt, tol, seeds, stats, u_prev=None):
    if dt <= 0.0:
        raise ValueError("dt must be positive")
    u = np.asarray(u, dtype=float)
    if scheme in ("rb_euler", "epi3"):
        J = _device_jacobian(problem, u)
        A = J.scaled(dt)
        fn = problem.rhs(u)
        if scheme == "rb_euler":
            return u + _engine(A, {1: dt * fn}, [1.0], tol, seeds, "rbe", stats)[:, 0]
        if u_prev is None:
            raise ValueError("epi3 requires the previous state")
        r = problem.rhs(u_prev) - fn - _matvec(J, u_prev - u)
        W = _engine(A, {1: dt * fn, 2: (2.0 / 3.0) * dt * r}, [1.0], tol, seeds,
                    "epi3", stats)
        return u + W[:, 0]
    if not np.all(np.isfinite(u)):
        raise ValueError("state must be finite")
    J = _device_jacobian(problem, u)
    fn = problem.rhs(u)

    def dev(U):
        return problem.rhs(U) - fn - _matvec(J, U - u)

    A = J.scaled(dt)
    v = dt * fn
    if scheme == "exprb42":
        W1 = _engine(A, {1: v}, [0.75], tol, seeds, "exprb42/1", stats)
        d2 = dev(u + W1[:, 0])
        W2 = _engine(A, {1: v, 3: (32.0 / 9.0) * dt * d2}, [1.0], tol, seeds,
                     "exprb42/2", stats)
        return u + W2[:, 0]
    if scheme == "pexprb43":
        W1 = _engine(A, {1: v}, [0.5, 1.0], tol, seeds, "pexprb43/1", stats)
        U2, U3 = u + W1[:, 0], u + W1[:, 1]
        d2, d3 = dev(U2), dev(U3)
        W2 = _engine(A, {3: dt * (16.0 * d2 - 2.0 * d3),
                         4: dt * (-48.0 * d2 + 12.0 * d3)}, [1.0], tol, seeds,
                     "pexprb43/2", stats)
        return U3 + W2[:, 0]
    W1 = _engine(A, {1: v}, [0.5, 0.9], tol, seeds, "exprb53/1", stats)
    d2 = dev(u + W1[:, 0])
    W2 = _engine(A, {3: dt * d2}, [0.5, 0.9], tol, seeds, "exprb53/2", stats)
    U3 = (u + W1[:, 1] + (27.0 / 25.0) * (W2[:, 0] / 0.5 ** 3)
          + (729.0 / 125.0) * (W2[:, 1] / 0.9 ** 3))
    d3 = dev(U3)
    W3 = _engine(A, {1: v, 3: dt * (18.0 * d2 - (250.0 / 81.0) * d3),
                     4: dt * (-60.0 * d2 + (500.0 / 27.0) * d3)}, [1.0], tol,
                 seeds, "exprb53/3", stats)
    return u + W3[:, 0]


def _step(problem, scheme, u_n, dt, tol, seeds, stats, u_prev=None):
    if getattr(problem, "ops", None) is not None:
        return _swe_step(problem, scheme, u_n, dt, tol, seeds, stats, u_prev)
    return _host_step(problem, scheme, u_n, dt, tol, seeds, stats, u_prev)


def step_rb_euler(problem, u_n, dt, tol=1e-4, seeds=None, stats=None):
    """Exponential Rosenbrock-Euler: u + dt*phi_1(dt J) F(u)."""
    return _step(problem, "rb_euler", u_n, dt, tol, seeds, stats)


def step_epi3(problem, u_n, u_prev, dt, tol=1e-4, seeds=None, stats=None):
    """Third-order exponential multistep step using one history state."""
    if u_prev is None:
        raise ValueError("epi3 requires the previous state")
    return _step(problem, "epi3", u_n, dt, tol, seeds, stats, u_prev)


def step_exprb42(problem, u_n, dt, tol=1e-4, seeds=None, stats=None):
    """Fourth-order two-stage scheme (node 3/4, phi_3 correction)."""
    return _step(problem, "exprb42", u_n, dt, tol, seeds, stats)


def step_pexprb43(problem, u_n, dt, tol=1e-4, seeds=None, stats=None):
    """Fourth-order scheme whose two stages share one engine call."""
    return _step(problem, "pexprb43", u_n, dt, tol, seeds, stats)


def step_exprb53(problem, u_n, dt, tol=1e-4, seeds=None, stats=None):
    """Fifth-order three-stage scheme (nodes 1/2 and 9/10)."""
    return _step(problem, "exprb53", u_n, dt, tol, seeds, stats)


def _integrate_swe(problem, scheme, u0, dt, t_end, tol, observers, keep_states):
    ctx = _swe.context(problem.ops)
    ctx.reset_seeds()
    u0 = np.asarray(u0, dtype=float)
    ctx.set_state(u0)
    ctx.set_prev(None)
    t = 0.0
    records = [StepRecord(t=0.0, u=u0.copy(), dt=0.0)]
    for obs in observers:
        obs(records[0])
    first = True
    while t < t_end - 1e-12 * max(t_end, 1.0):
        h = min(dt, t_end - t)
        sch = "rb_euler" if (scheme == "epi3" and first) else scheme
        calls = ctx.step(sch, h, tol)
        first = False
        t += h
        need = keep_states or observers
        rec = StepRecord(t=t, u=ctx.get_state() if need else None, dt=h,
                         matvecs=sum(int(c.matvecs) for c in calls),
                         substeps=sum(int(c.substeps) for c in calls))
        records.append(rec)
        for obs in observers:
            obs(rec)
    if not keep_states:
        records[-1].u = ctx.get_state()
    return records


def integrate(problem, scheme, u0, dt, t_end, tol=1e-4, observers=(),
              keep_states=True):
    """Fixed-step trajectory with warm-started engine seeds
    (integrators.py:318-369).  ``keep_states=False`` (shallow-water route)
    skips the per-step host copy except for the final state."""
    if scheme not in SCHEME_NAMES:
        raise ValueError(f"unknown scheme {scheme!r}")
    if dt <= 0.0:
        raise ValueError("dt must be positive")
    if getattr(problem, "ops", None) is not None:
        return _integrate_swe(problem, scheme, u0, dt, t_end, tol, observers,
                              keep_states)
    u = np.asarray(u0, dtype=float).copy()
    t = 0.0
    seeds = EngineSeeds()
    stats = _StepStats()
    records = [StepRecord(t=0.0, u=u.copy(), dt=0.0)]
    for obs in observers:
        obs(records[0])
    u_prev = None
    while t < t_end - 1e-12 * max(t_end, 1.0):
        h = min(dt, t_end - t)
        m0, s0 = stats.matvecs, stats.substeps
        if scheme == "epi3":
            if u_prev is None:
                u_next = _host_step(problem, "rb_euler", u, h, tol, seeds, stats)
            else:
                u_next = _host_step(problem, "epi3", u, h, tol, seeds, stats, u_prev)
            u_prev = u
        else:
            u_next = _host_step(problem, scheme, u, h, tol, seeds, stats)
        t += h
        u = u_next
        rec = StepRecord(t=t, u=u.copy(), dt=h, matvecs=stats.matvecs - m0,
                         substeps=stats.substeps - s0)
        records.append(rec)
        for obs in observers:
            obs(rec)
    return records
