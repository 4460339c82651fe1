"""Every BASELINE config at its stated length against the reference itself
(fixtures from tests/golden/make_long_golden.py, run on the CPU with the
unmodified reference): C1 pEXPRB4 over one day at dt = 900/1800/3600/7200 s,
C2 EXPRB5 240 x 1800 s (5 days), C3 EXPRB4 and EPI3 144 x 600 s (1 day),
C4 at L9 EXPRB4 and EXPRB5 10 x 900 s.

Bar (BASELINE.json north_star): every engine call's substeps, rejections,
matvecs and final Krylov dimension identical to the reference's, and the
relative L2 state difference <= 1e-9 -- checked on the WHOLE state at every
checkpoint (1, 2, 4, ..., final) through a CountSketch of each field
(tests/golden/sketch.py; a linear map, so sketch(u) - sketch(ref) =
sketch(u - ref), whose norm estimates ||u - ref|| within a few percent),
plus 1024-4096 sampled entries and the per-field norms of every step.
"""

import glob
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

from sketch import field_norms, sketch_rel  # noqa: E402

from paper_1805_02144_b200 import swe as gswe  # noqa: E402
from paper_1805_02144_b200.states import make_config  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = 1e-9
FIXTURES = sorted(glob.glob(os.path.join(HERE, "golden", "long_*.npz")))


def _ids(p):
    return os.path.basename(p)[5:-4]


def digest(ops):
    import hashlib
    h = hashlib.sha256()
    for name in ("Gx", "Gy", "Gz", "Dx", "Dy", "Dz", "Vx", "Vy", "Vz", "L", "Df"):
        c = getattr(ops, name).csr
        h.update(np.ascontiguousarray(c.indptr).tobytes())
        h.update(np.ascontiguousarray(c.indices).tobytes())
        h.update(np.ascontiguousarray(c.data).tobytes())
    for f in ("n_x", "n_y", "n_z", "f", "h_s"):
        h.update(np.ascontiguousarray(getattr(ops, f)).tobytes())
    return h.hexdigest()


def _level(path):
    name = os.path.basename(path)
    tag = name.split("_")[1]
    return int(tag.split("l")[1]) if "l" in tag[1:] else None


@pytest.mark.parametrize("path", FIXTURES, ids=[_ids(p) for p in FIXTURES])
def test_config_full_length_matches_reference(path):
    g = np.load(path)
    cfg, scheme = str(g["cfg"]), str(g["scheme"])
    dt, nsteps, tol = float(g["dt"]), int(g["nsteps"]), float(g["tol"])
    ops, u0, _ = make_config(cfg, _level(path))
    assert digest(ops) == str(g["digest"]), "grid/state generator changed"
    ctx = gswe.SweContext(ops)
    ctx.set_state(u0)
    ctx.set_prev(None)
    ctx.reset_seeds()
    ref_calls = g["calls"]  # step, p, substeps, rejections, matvecs, m_final, tau_final
    cps = [int(c) for c in g["checkpoints"]]
    idx = g["sample_idx"]
    worst = 0.0
    ci = 0
    for k in range(1, nsteps + 1):
        sch = "rb_euler" if (scheme == "epi3" and k == 1) else scheme
        cs = ctx.step(sch, dt, tol)
        mine = [(int(c.substeps), int(c.rejections), int(c.matvecs), int(c.m_final))
                for c in cs if not c.skipped]
        theirs = [tuple(int(x) for x in r[2:6]) for r in ref_calls if int(r[0]) == k]
        assert mine == theirs, (
            f"{cfg} {scheme} dt={dt:g}: engine decisions differ at step {k}: "
            f"device (substeps, rejections, matvecs, m) {mine} vs reference {theirs}")
        if k in cps:
            u = ctx.get_state()
            fn = field_norms(u)
            ref_fn = g["field_norms"][k - 1]
            assert np.all(np.abs(fn - ref_fn) <= TOL * ref_fn + 1e-300), (k, fn, ref_fn)
            ref_norm = float(np.linalg.norm(ref_fn))
            est, _ = sketch_rel(u, g["sketches"][ci], ref_norm)
            worst = max(worst, est)
            assert est <= TOL, f"step {k}: sketched full-state rel L2 {est:.3e}"
            samp = g["final_sample"] if k == nsteps else g["cp_samples"][ci]
            sel = idx if k == nsteps else idx[:samp.shape[0]]
            assert np.max(np.abs(u[sel] - samp)) <= TOL * np.max(np.abs(samp))
            ci += 1
    assert ci == len(cps)
    print(f"{_ids(path)}: {nsteps} steps, worst sketched rel L2 {worst:.2e}")


def test_c4_l10_runs_conserve_mass():
    """C4 at L10 (10.5 M cells): the reference oracle is not run (its
    assembled Jacobian alone needs >60 GB of host RAM), so
    parity is not pinned at L10.  What is checked on the device: 10 EXPRB4
    steps complete, the state stays finite and the total mass (h weighted by
    cell area) is conserved to 1e-12 (the divergence operator is
    conservative, Df's Laplacian rows sum to zero)."""
    if not os.environ.get("EIK_RUN_L10"):
        pytest.skip("L10 run is opt-in (EIK_RUN_L10=1): building the 10.5 M-cell grid "
                    "takes ~3 min of host time")
    ops, u0, spec = make_config("C4", 10)
    ctx = gswe.context(ops)  # the context diagnostics() reads
    ctx.set_state(u0)
    ctx.reset_seeds()
    m0 = gswe.diagnostics(ops, area_weighted=True).mass
    for _ in range(spec.steps):
        ctx.step("exprb42", spec.dt, spec.tol)
    m1 = gswe.diagnostics(ops, area_weighted=True).mass
    assert np.all(np.isfinite(ctx.get_state()))
    assert abs(m1 - m0) <= 1e-12 * abs(m0)


@pytest.mark.skip(reason="C4 at L10: oracle not run (RAM) -- the reference's assembled "
                         "4N x 4N Jacobian and its J assembly need more than the 62 GB of "
                         "host memory available where fixtures are made (SURVEY.md §8d)")
def test_c4_l10_matches_reference():
    pass
