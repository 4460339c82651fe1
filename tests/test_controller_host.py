"""The device controller's scalar logic (csrc/eik_control.h), compiled for
the host, against the oracle restatement of phipm.py:217-313."""

import ctypes as C
import math
import os
import subprocess

import numpy as np
import pytest

from oracle.expint_oracle import adapt_step, cost_model

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def ctl(tmp_path_factory):
    out = tmp_path_factory.mktemp("ctl") / "libctl.so"
    src = os.path.join(HERE, "host", "control_harness.cpp")
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", str(out), src],
                   check=True)
    lib = C.CDLL(str(out))
    D, L = C.c_double, C.c_longlong
    lib.t_cost.restype = D
    lib.t_cost.argtypes = [D, L, L, L, L, D, D, D]
    lib.t_adapt.restype = None
    lib.t_adapt.argtypes = [D, L, D, D, D, D, D, L, D, D, L, L, L,
                            C.POINTER(D), C.POINTER(L)]
    lib.t_init.argtypes = [D, L, D, D, L, L, C.POINTER(D), C.POINTER(L)]
    lib.t_powfact.restype = D
    lib.t_powfact.argtypes = [D, C.c_int]
    return lib


def test_cost_matches_oracle(ctl):
    rng = np.random.default_rng(3)
    for _ in range(2000):
        tau = float(10 ** rng.uniform(-4, 0))
        m = int(rng.integers(1, 101))
        N = int(rng.integers(10, 50_000_000))
        nA = int(rng.integers(N, 12 * N))
        p = int(rng.integers(0, 5))
        nh = float(10 ** rng.uniform(-3, 3))
        t_k = float(rng.uniform(0, 1))
        t_out = float(rng.uniform(0, 1))
        assert ctl.t_cost(tau, m, N, nA, p, nh, t_out, t_k) == \
            cost_model(tau, m, N, nA, p, nh, t_out, t_k)
    # SPEC.md:187 example as the code computes it
    assert ctl.t_cost(0.1, 10, 100, 500, 2, 1.0, 1.0, 0.0) == \
        cost_model(0.1, 10, 100, 500, 2, 1.0, 1.0, 0.0)


def test_adapt_matches_oracle(ctl):
    rng = np.random.default_rng(4)
    D, L = C.c_double, C.c_longlong
    hit = {"tau": 0, "m": 0, "crawl": 0, "zero": 0}
    for k in range(5000):
        tau = float(10 ** rng.uniform(-3, 0))
        m = int(rng.integers(1, 101))
        t_k = float(rng.uniform(0, 0.9))
        t_out = float(min(1.0, t_k + rng.uniform(0.01, 1.0)))
        eps = 0.0 if k % 50 == 0 else float(10 ** rng.uniform(-14, -2))
        nh = float(10 ** rng.uniform(-2, 2.5))
        p = int(rng.integers(0, 5))
        tol = float(10 ** rng.uniform(-10, -4))
        N = int(rng.integers(100, 10_000_000))
        nA = int(40 * N)
        want = adapt_step(tau, m, t_k, eps, nh, t_out, 1.0, p, tol, 1.4, 100, N, nA)
        to, mo = D(), L()
        ctl.t_adapt(tau, m, t_k, eps, nh, t_out, 1.0, p, tol, 1.4, 100, N, nA,
                    C.byref(to), C.byref(mo))
        assert (to.value, mo.value) == want
        hit["zero" if eps == 0 else ("m" if mo.value != m else "tau")] += 1
    assert min(hit["tau"], hit["m"], hit["zero"]) > 0


def test_initial_tau_m(ctl):
    D, L = C.c_double, C.c_longlong
    cases = [(-1.0, 1, 0.75, 0.75, 100, 10248), (1e-9, 7, 0.5, 1.0, 100, 10248),
             (0.3, 400, 0.5, 0.9, 100, 40), (2.0, 0, 1.0, 1.0, 100, 10)]
    for tau_init, m_init, r0, rl, mmax, n in cases:
        # phipm.py:300-313
        mcap = min(mmax, n)
        tau = tau_init if tau_init > 0 else r0
        tau = min(max(tau, rl / (10.0 * 100)), r0)
        m = min(max(m_init, 1), mcap)
        to, mo = D(), L()
        ctl.t_init(tau_init, m_init, r0, rl, mmax, n, C.byref(to), C.byref(mo))
        assert (to.value, mo.value) == (tau, m)


def test_pow_over_factorial(ctl):
    for t in (0.0, 0.37, 0.5, 0.9, 1.0):
        for ell in range(6):
            assert ctl.t_powfact(t, ell) == t ** ell / math.factorial(ell)


def test_shared_reciprocal_division_is_exact(tmp_path):
    """form_x's x / h through one shared reciprocal and two FMAs (the tiled
    pass, csrc/eik_dev.cuh) gives the bits of IEEE division."""
    try:
        if " fma " not in open("/proc/cpuinfo").read().replace("\n", " "):
            pytest.skip("host CPU without FMA")
    except OSError:
        pass
    exe = tmp_path / "shared_div"
    subprocess.run(["gcc", "-O2", "-mfma", "-ffp-contract=off", "-o", str(exe),
                    os.path.join(HERE, "host", "shared_div.c"), "-lm"], check=True)
    out = subprocess.run([str(exe), "20000000"], check=True, capture_output=True, text=True)
    assert int(out.stdout.strip()) == 0
