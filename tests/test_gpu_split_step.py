"""The split step graph (k_swe_cont / k_swe_sweep under a conditional while
node, the default) against the monolithic step kernel (EIK_STEP_MONO=1):
bitwise-identical states and identical per-call counters for every scheme,
and the device-side kernel count."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, %r)
from paper_1805_02144_b200.states import make_config
from paper_1805_02144_b200 import swe as gswe
out = {}
for scheme, cfg, steps in (("exprb42", "C0", 3), ("pexprb43", "C0", 2), ("exprb53", "C0", 2),
                           ("epi3", "C0", 3), ("exprb42", "C3", 2)):
    ops, u0, spec = make_config(cfg)
    ctx = gswe.SweContext(ops)
    ctx.set_state(u0)
    if scheme == "epi3":
        ctx.set_prev(u0)
    calls = []
    k0 = ctx.launches()
    for _ in range(steps):
        infos = ctx.step(scheme, spec.dt, spec.tol)
        calls.append([(c.matvecs, c.substeps, c.rejections, c.attempts, c.m_final, c.tau_final)
                      for c in infos])
    u = ctx.get_state()
    out[scheme + cfg] = {"u": u.tobytes().hex(), "calls": calls,
                         "launches": ctx.launches() - k0}
print(json.dumps(out))
"""


def _run(mono, host=False, extra=None):
    env = dict(os.environ)
    for k in ("EIK_STEP_MONO", "EIK_STEP_HOST", "EIK_SORT_HALO",
              "EIK_TILES_EXTRA"):
        env.pop(k, None)
    env.update(extra or {})
    if mono:
        env["EIK_STEP_MONO"] = "1"
    if host:
        env["EIK_STEP_HOST"] = "1"
    r = subprocess.run([sys.executable, "-c", _SCRIPT % ROOT], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_split_step_matches_monolithic_bitwise():
    split, mono = _run(False), _run(True)
    assert split.keys() == mono.keys()
    for k in split:
        assert split[k]["calls"] == mono[k]["calls"], k
        assert split[k]["u"] == mono[k]["u"], k
        u = np.frombuffer(bytes.fromhex(split[k]["u"]), dtype=np.float64)
        assert np.all(np.isfinite(u))
        # monolithic: one graph launch per step; split: at least one k_swe_cont
        # per step plus a k_swe_sweep + k_swe_cont pair per tiled sweep
        nsteps = len(split[k]["calls"])
        assert mono[k]["launches"] >= nsteps
        assert split[k]["launches"] >= mono[k]["launches"] + 2 * nsteps


def test_hostloop_matches_graph_bitwise():
    """Host-loop mode (kernel-by-kernel launches, used for the sweep roofline
    and ncu) runs exactly the graph's kernels: same bits, same counters."""
    graph, host = _run(False), _run(False, host=True)
    for k in graph:
        assert graph[k]["calls"] == host[k]["calls"], k
        assert graph[k]["u"] == host[k]["u"], k


def test_layout_knobs_do_not_change_results():
    """The device layout choices made at context creation are labels only:
    halo rings sorted by device index (EIK_SORT_HALO=1) give the same bits and
    counters as the default layout."""
    base = _run(False)
    for extra in ({"EIK_SORT_HALO": "1"},):
        other = _run(False, extra=extra)
        for k in base:
            assert base[k]["calls"] == other[k]["calls"], (extra, k)
            assert base[k]["u"] == other[k]["u"], (extra, k)
