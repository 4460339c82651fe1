"""Oracle restatement of the phipm/IOM2 engine and the exponential schemes.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The arithmetic follows
the reference operation by operation (same numpy calls, same order) so that
the restatement reproduces the reference bit for bit; the structure is our
own.  Citations are to /root/reference/pkg/src/expintkit/.
"""

import math

import numpy as np

# kernels.py:20-31
_CAP = 256
_THETA13 = 5.37
_B13 = (64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
        1187353796428800.0, 129060195264000.0, 10559470521600.0,
        670442572800.0, 33522128640.0, 1323241920.0, 40840800.0,
        960960.0, 16380.0, 182.0, 1.0)
# krylov.py:17, phipm.py:28-31
_BREAKDOWN = 1e-14
MAX_ATTEMPTS = 10 ** 6
_CRAWL = 100


class PhipmFailureOracle(RuntimeError):
    """phipm.py:34-42."""

    def __init__(self, msg, t_reached, substeps, rejections, matvecs):
        super().__init__(msg)
        self.t_reached = t_reached
        self.substeps = substeps
        self.rejections = rejections
        self.matvecs = matvecs


class OracleOperator:
    """A matvec plus (n, nnz) with a performed-product counter
    (phipm.py:45-70)."""

    def __init__(self, matvec, n, nnz):
        self._mv = matvec
        self.n = n
        self.nnz = nnz
        self.count = 0

    def __call__(self, x):
        self.count += 1
        return self._mv(x)

    @classmethod
    def from_matrix(cls, A):
        """phipm.py:73-84 for ndarray / scipy / objects with .csr."""
        import scipy.sparse
        if hasattr(A, "csr"):
            A = A.csr
        if scipy.sparse.issparse(A):
            c = A.tocsr()
            return cls(c.dot, c.shape[0], c.nnz)
        A = np.asarray(A, dtype=float)
        return cls(A.dot, A.shape[0], int(np.count_nonzero(A)))


# ---------------------------------------------------------------- dense part

def expm_pade13(H):
    """kernels.py:119-145: degree-13 Pade, s = ceil(log2(|H|_1/5.37))_+."""
    H = np.asarray(H, dtype=float)
    n = H.shape[0]
    nrm = np.linalg.norm(H, 1) if n else 0.0
    s = max(0, int(math.ceil(math.log2(nrm / _THETA13)))) if nrm > _THETA13 else 0
    X = H / (2.0 ** s)
    b = _B13
    eye = np.eye(n)
    X2 = X @ X
    X4 = X2 @ X2
    X6 = X2 @ X4
    odd = X @ (X6 @ (b[13] * X6 + b[11] * X4 + b[9] * X2)
               + b[7] * X6 + b[5] * X4 + b[3] * X2 + b[1] * eye)
    even = (X6 @ (b[12] * X6 + b[10] * X4 + b[8] * X2)
            + b[6] * X6 + b[4] * X4 + b[2] * X2 + b[0] * eye)
    E = np.linalg.solve(even - odd, even + odd)
    for _ in range(s):
        E = E @ E
    return E


def augment(H, p):
    """kernels.py:148-172."""
    m = H.shape[0]
    dim = m + p + 1
    if dim > _CAP:
        raise ValueError(f"augmented dense size {dim} exceeds cap {_CAP}")
    Hh = np.zeros((dim, dim))
    Hh[:m, :m] = H
    if m > 0:
        Hh[0, m] = 1.0
    for j in range(p):
        Hh[m + j, m + j + 1] = 1.0
    return Hh


def phi_columns_aug(H, tau, p):
    """kernels.py:175-193: [e^{tH}e1, t^j phi_j(tH) e1 for j=1..p+1]."""
    m = H.shape[0]
    E = expm_pade13(tau * augment(H, p))
    return [E[:m, 0].copy()] + [E[:m, m + j - 1].copy() for j in range(1, p + 2)]


# ------------------------------------------------------------- Krylov part

class Decomp:
    """krylov.py:20-40 (V, H, h_next, v_next, beta, breakdown)."""

    __slots__ = ("V", "H", "h_next", "v_next", "beta", "breakdown")

    def __init__(self, V, H, h_next, v_next, beta, breakdown):
        self.V, self.H, self.h_next = V, H, h_next
        self.v_next, self.beta, self.breakdown = v_next, beta, breakdown


def iom_arnoldi(matvec, w, m, iom=2):
    """krylov.py:53-112: Arnoldi with MGS against the last ``iom`` vectors;
    the basis is stored n x m C-order exactly like the reference (so BLAS
    sees the same strided columns)."""
    beta = np.linalg.norm(w)
    if beta == 0.0:
        raise ValueError("seed vector must be nonzero")
    n = w.shape[0]
    V = np.zeros((n, m))
    H = np.zeros((m, m))
    V[:, 0] = w / beta
    h_next, v_next, broke, keep = 0.0, None, False, m
    for j in range(m):
        z = matvec(V[:, j])
        for i in range(max(0, j - iom + 1), j + 1):
            c = V[:, i] @ z
            H[i, j] = c
            z = z - c * V[:, i]
        h = np.linalg.norm(z)
        if h < _BREAKDOWN * beta:
            broke, keep, h_next, v_next = True, j + 1, 0.0, None
            break
        if j + 1 < m:
            H[j + 1, j] = h
            V[:, j + 1] = z / h
        else:
            h_next, v_next = h, z / h
    if broke and keep < m:
        V, H = V[:, :keep], H[:keep, :keep]
    return Decomp(V, H, h_next, v_next, beta, broke)


def krylov_apply(dec, tau, p):
    """krylov.py:115-146: (phi_p approximation with the correction term,
    eps_m)."""
    cols = phi_columns_aug(dec.H, tau, p)
    m = dec.H.shape[0]
    approx = dec.beta * (dec.V @ (cols[p] / tau ** p))
    if dec.breakdown or dec.v_next is None:
        return approx, 0.0
    corner = cols[p + 1][m - 1]
    approx = approx + (dec.beta * dec.h_next * (corner / tau ** p) * dec.v_next)
    return approx, dec.beta * abs(dec.h_next) * abs(corner)


# ------------------------------------------------------------ engine logic

def cost_model(tau, m, N, n_A, p, norm_hhat, t_out, t_k):
    """phipm.py:217-238 (whole bracket times the substep count)."""
    if tau <= 0.0:
        raise ValueError("tau must be positive")
    M = 44.0 / 3.0
    if norm_hhat > _THETA13:
        M += 2.0 * math.ceil(math.log2(norm_hhat / _THETA13))
    k = math.ceil((t_out - t_k) / tau) if t_out > t_k else 1
    return k * (m * (N + n_A) + 2 * max(p - 1, 0) * (n_A + N)
                + M * (m + p + 1) ** 3 + (2 * p + 1) * N)


def adapt_step(tau, m, t_k, eps, norm_hhat, t_out, horizon, p, tol, delta,
               m_max, N, n_A):
    """phipm.py:241-288 -> (tau_new, m_new)."""
    remaining = max(horizon - t_k, tau * 1e-16)
    omega = t_out * eps / (tau * tol)
    if omega == 0.0:
        return min(2.0 * tau, remaining), m
    tau_pred = tau * omega ** (-1.0 / (p + 1))
    tau_cand = min(max(tau_pred, tau / 5.0), 2.0 * tau, remaining)
    m_cap = min(m_max, N)
    if remaining / tau_cand > _CRAWL and m < m_cap:
        return tau_cand, m_cap
    if omega > delta:
        m_cand = m + int(math.ceil(math.log2(max(omega, 1.0))))
    else:
        m_cand = m - 1
    m_cand = min(max(m_cand, 1), m_cap)
    if m_cand == m:
        return tau_cand, m
    c_tau = cost_model(max(tau_pred, 1e-16), m, N, n_A, p,
                       norm_hhat * tau_pred / tau if tau > 0 else 0.0,
                       t_out, t_k)
    c_m = cost_model(tau, m_cand, N, n_A, p, norm_hhat, t_out, t_k)
    return (tau_cand, m) if c_tau <= c_m else (tau, m_cand)


class EngineResult:
    __slots__ = ("W", "substeps", "rejections", "matvecs", "tau_final",
                 "m_final", "trace")

    def __init__(self, **kw):
        for k, v in kw.items():
            setattr(self, k, v)


def _w_recurrence(op, y, vs, t, zero_skip):
    """phipm.py:159-182."""
    p = len(vs) - 1
    ws = [np.asarray(y, dtype=float)]
    for j in range(1, p + 1):
        prev = ws[-1]
        acc = np.zeros_like(prev) if (zero_skip and not prev.any()) else op(prev)
        for ell in range(p - j + 1):
            v = vs[j + ell]
            if v.any():
                acc = acc + (t ** ell / math.factorial(ell)) * v
        ws.append(acc)
    return ws


def _advance(op, ws, tau, m_req, iom_req):
    """phipm.py:185-214 -> (cand, eps, norm_hhat)."""
    p = len(ws) - 1
    cand = np.zeros_like(ws[0])
    for j in range(p):
        cand = cand + (tau ** j / math.factorial(j)) * ws[j]
    wp = ws[p]
    if not wp.any():
        return cand, 0.0, 0.0
    n = wp.shape[0]
    m = min(m_req, n)
    dec = iom_arnoldi(op, wp, m, iom=iom_req if m < n else n)
    approx, eps = krylov_apply(dec, tau, p)
    cand = cand + tau ** p * approx
    return cand, eps, tau * np.linalg.norm(augment(dec.H, p), 1)


def engine_run(op, vs, rho, tol=1e-4, m_init=1, iom=2, m_max=100, delta=1.4,
               tau_init=None, zero_skip=True, trace=False,
               max_attempts=None):
    """phipm.py:291-370: y(rho_i) = sum_l rho_i^l phi_l(rho_i A) v_l."""
    if not isinstance(op, OracleOperator):
        op = OracleOperator.from_matrix(op)
    vs = [np.asarray(v, dtype=float) for v in vs]
    n = vs[0].shape[0]
    p = len(vs) - 1
    rho = [float(r) for r in rho]
    limit = MAX_ATTEMPTS if max_attempts is None else max_attempts
    m_cap = min(m_max, n)
    y = vs[0].copy()
    t = 0.0
    tau = tau_init if tau_init else rho[0]
    m = min(max(m_init, 1), m_cap)
    tau = min(max(tau, rho[-1] / (10.0 * _CRAWL)), rho[0])
    W = np.zeros((n, len(rho)))
    log = []
    acc_n = rej_n = tries = 0
    for col, t_out in enumerate(rho):
        while t < t_out:
            tries += 1
            if tries > limit:
                raise PhipmFailureOracle(
                    f"no convergence within {limit} substeps "
                    f"(t reached {t:.3e} of {t_out:.3e})",
                    t_reached=t, substeps=acc_n, rejections=rej_n,
                    matvecs=op.count)
            tau_nom = tau
            lands = t + tau >= t_out
            if lands:
                tau = t_out - t
            ws = _w_recurrence(op, y, vs, t, zero_skip)
            cand, eps, nh = _advance(op, ws, tau, m, iom)
            omega = t_out * eps / (tau * tol)
            ok = omega <= delta
            if trace:
                log.append((tries, t, tau, m, eps, omega, ok))
            tau_new, m_new = adapt_step(tau, m, t, eps, nh, t_out, rho[-1], p,
                                        tol, delta, m_max, n, op.nnz)
            if ok:
                y = cand
                t = t_out if lands else t + tau
                acc_n += 1
                if lands:
                    tau_new = max(tau_new, tau_nom)
            else:
                rej_n += 1
            tau = max(tau_new, 1e-16)
            m = min(max(m_new, 1), m_cap)
        W[:, col] = y
    return EngineResult(W=W, substeps=acc_n, rejections=rej_n,
                        matvecs=op.count, tau_final=tau, m_final=m, trace=log)


# ------------------------------------------------------------ the schemes

class OracleSeeds:
    """integrators.py:73-83: warm start (tau_final, m_final) per slot."""

    def __init__(self):
        self.table = {}

    def get(self, slot):
        return self.table.get(slot, (None, 1))

    def put(self, slot, res):
        self.table[slot] = (res.tau_final, res.m_final)


class CallLog:
    """Per-engine-call counters (what the GPU trace is compared with)."""

    def __init__(self):
        self.calls = []

    def add(self, slot, res):
        self.calls.append((slot, res.substeps, res.rejections, res.matvecs,
                           res.m_final, res.tau_final))


def _call(J_op, dt, vecs, rho, tol, seeds, slot, log):
    """integrators.py:115-137: p = max index, zero padding, all-zero
    short-cut, A x = dt * (J x) scaled after the product."""
    p = max(vecs)
    n = next(iter(vecs.values())).shape[0]
    vs = [vecs.get(k, np.zeros(n)) for k in range(p + 1)]
    if not any(v.any() for v in vs):
        return np.zeros((n, len(rho)))
    op = OracleOperator(lambda x: dt * J_op.matvec(x), J_op.n_rows, J_op.nnz)
    tau0, m0 = seeds.get(slot)
    res = engine_run(op, vs, rho, tol=tol, m_init=m0, tau_init=tau0)
    seeds.put(slot, res)
    if log is not None:
        log.add(slot, res)
    return res.W


def _rhs(problem, u):
    out = np.asarray(problem.f(u), dtype=float)
    if not np.all(np.isfinite(out)):
        raise ValueError("non-finite right-hand side")
    return out


def step_oracle(problem, scheme, u, dt, tol, seeds, log=None, u_prev=None):
    """integrators.py:140-224 (problem has .f(u) and .jac(u) -> matrix with
    .matvec/.n_rows/.nnz)."""
    u = np.asarray(u, dtype=float)
    if scheme in ("rb_euler", "epi3"):
        J = problem.jac(u)
        fn = _rhs(problem, u)
        if scheme == "rb_euler":
            W = _call(J, dt, {1: dt * fn}, [1.0], tol, seeds, "rbe", log)
            return u + W[:, 0]
        r = _rhs(problem, u_prev) - fn - J.matvec(u_prev - u)
        W = _call(J, dt, {1: dt * fn, 2: (2.0 / 3.0) * dt * r}, [1.0], tol,
                  seeds, "epi3", log)
        return u + W[:, 0]
    if not np.all(np.isfinite(u)):
        raise ValueError("state must be finite")
    J = problem.jac(u)
    fn = _rhs(problem, u)

    def dev(U):  # integrators.py:101-102
        return _rhs(problem, U) - fn - J.matvec(U - u)

    v = dt * fn
    if scheme == "exprb42":
        W1 = _call(J, dt, {1: v}, [0.75], tol, seeds, "exprb42/1", log)
        d2 = dev(u + W1[:, 0])
        W2 = _call(J, dt, {1: v, 3: (32.0 / 9.0) * dt * d2}, [1.0], tol,
                   seeds, "exprb42/2", log)
        return u + W2[:, 0]
    if scheme == "pexprb43":
        W1 = _call(J, dt, {1: v}, [0.5, 1.0], tol, seeds, "pexprb43/1", log)
        U2 = u + W1[:, 0]
        U3 = u + W1[:, 1]
        d2, d3 = dev(U2), dev(U3)
        W2 = _call(J, dt, {3: dt * (16.0 * d2 - 2.0 * d3),
                           4: dt * (-48.0 * d2 + 12.0 * d3)},
                   [1.0], tol, seeds, "pexprb43/2", log)
        return U3 + W2[:, 0]
    if scheme == "exprb53":
        W1 = _call(J, dt, {1: v}, [0.5, 0.9], tol, seeds, "exprb53/1", log)
        d2 = dev(u + W1[:, 0])
        W2 = _call(J, dt, {3: dt * d2}, [0.5, 0.9], tol, seeds, "exprb53/2", log)
        U3 = (u + W1[:, 1] + (27.0 / 25.0) * (W2[:, 0] / 0.5 ** 3)
              + (729.0 / 125.0) * (W2[:, 1] / 0.9 ** 3))
        d3 = dev(U3)
        W3 = _call(J, dt, {1: v, 3: dt * (18.0 * d2 - (250.0 / 81.0) * d3),
                           4: dt * (-60.0 * d2 + (500.0 / 27.0) * d3)},
                   [1.0], tol, seeds, "exprb53/3", log)
        return u + W3[:, 0]
    raise ValueError(f"unknown scheme {scheme!r}")


def integrate_oracle(problem, scheme, u0, dt, t_end, tol=1e-4, log=None,
                     keep_states=False):
    """integrators.py:318-369 -> (final state, per-step (matvecs, substeps),
    optional list of states)."""
    u = np.asarray(u0, dtype=float).copy()
    t = 0.0
    seeds = OracleSeeds()
    u_prev = None
    per_step, states = [], [u.copy()] if keep_states else None
    log = CallLog() if log is None else log
    while t < t_end - 1e-12 * max(t_end, 1.0):
        h = min(dt, t_end - t)
        k0 = len(log.calls)
        if scheme == "epi3" and u_prev is None:
            nxt = step_oracle(problem, "rb_euler", u, h, tol, seeds, log)
        else:
            nxt = step_oracle(problem, scheme, u, h, tol, seeds, log, u_prev)
        if scheme == "epi3":
            u_prev = u
        new = log.calls[k0:]
        per_step.append((sum(c[3] for c in new), sum(c[1] for c in new)))
        t += h
        u = nxt
        if keep_states:
            states.append(u.copy())
    return u, per_step, states, log
