"""State sketches for long-run parity fixtures (test infrastructure).

A full fp64 state at L8/L9 is 21-84 MB, too large to commit for every
checkpoint of a 144-step run.  The fixtures therefore hold, per checkpoint,
a CountSketch of each field: K buckets, bucket b(i) and sign s(i) drawn from
a fixed seed, S_f(u)[k] = sum_{b(i)=k} s(i) u_f[i].  S is linear, so
S(u) - S(ref) = S(u - ref), and E||S d||^2 = ||d||^2 with a relative standard
deviation of about sqrt(2/K) (4.4 % at K = 1024 per field).  The full-state
relative L2 difference is estimated as
    sqrt(sum_f ||S_f(u) - S_f(ref)||^2) / ||ref||
with ||ref|| stored exactly, so the 1e-9 gate is checked on every entry of
the state, not on a sample.  Explicitly sampled entries are stored as well.
"""

import numpy as np

K = 1024
SEED = 20261020


def _hash(n_g):
    rng = np.random.default_rng(SEED + n_g)
    b = rng.integers(0, K, n_g)
    s = rng.integers(0, 2, n_g).astype(np.float64) * 2.0 - 1.0
    return b, s


_CACHE = {}


def sketch(u):
    """(4, K) CountSketch of the state [u_x; u_y; u_z; h]."""
    u = np.asarray(u, dtype=np.float64)
    n_g = u.shape[0] // 4
    if n_g not in _CACHE:
        _CACHE.clear()
        _CACHE[n_g] = _hash(n_g)
    b, s = _CACHE[n_g]
    return np.stack([np.bincount(b, weights=s * f, minlength=K) for f in np.split(u, 4)])


def field_norms(u):
    return np.array([np.linalg.norm(f) for f in np.split(np.asarray(u), 4)])


def sample_idx(n, count, seed=12345):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, size=min(count, n), replace=False))


def sketch_rel(u, sk_ref, norm_ref):
    """Estimated full-state relative L2 difference of ``u`` against the
    sketched reference, plus the (4,) per-field estimates of ||d_f||."""
    d = sketch(u) - sk_ref
    per = np.sqrt(np.sum(d * d, axis=1))
    return float(np.sqrt(np.sum(per ** 2)) / norm_ref), per
