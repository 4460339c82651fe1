"""Seeded initial states for BASELINE.json's five configurations.

The Williamson/Galewsky documents the paper uses (PAPER.md:1050-1059,
1528-1536) are not in the container; BASELINE.json's own text is the spec,
restated here.  Every generator draws from ``np.random.default_rng(seed)``
(the reference's RNG idiom, harness.py:108, 315) and returns the stacked
state ``[u_x; u_y; u_z; h]`` (swe.py:124-133) plus, where the config has
orography, a surface height ``h_s``.  ``h`` is the layer thickness: the
reference's energy uses ``g (h + h_s)`` (swe.py:161).

Choices BASELINE.json leaves open (recorded in DESIGN.md):
* C0/C1/C4 perturbation uses real spherical harmonics of degree 1..8;
* C1's wavenumber-4 stream function is the degree-5 pattern
  psi = -a^2 K cos^4(lat) sin(lat) cos(4 lon) with K set so max|zeta| = 8e-6;
  the height stays balanced to the zonal part only;
* C2 seed 3, centre latitude in [-45, 45] deg; C3 seed 4, jet profile
  u = u_max exp(-((lat - lat0)/10deg)^2), mean depth 10 km.
"""

from dataclasses import dataclass

import numpy as np
from scipy.special import sph_harm_y

from .grid import EARTH_OMEGA, EARTH_RADIUS, GRAVITY


@dataclass
class ConfigSpec:
    name: str
    level: int
    scheme: str
    dt: float
    steps: int
    tol: float
    seed: int


CONFIGS = {
    "C0": ConfigSpec("C0", 4, "exprb42", 3600.0, 24, 1e-8, 0),
    "C1": ConfigSpec("C1", 6, "pexprb43", 1800.0, 48, 1e-8, 1),
    "C2": ConfigSpec("C2", 7, "exprb53", 1800.0, 240, 1e-8, 3),
    "C3": ConfigSpec("C3", 8, "exprb42", 600.0, 144, 1e-8, 4),
    "C4": ConfigSpec("C4", 9, "exprb42", 900.0, 10, 1e-8, 2),
}


def _latlon(x):
    lat = np.arcsin(np.clip(x[:, 2], -1.0, 1.0))
    lon = np.arctan2(x[:, 1], x[:, 0])
    return lat, lon


def _zonal_unit(lon):
    return np.stack([-np.sin(lon), np.cos(lon), np.zeros_like(lon)], 1)


def _merid_unit(lat, lon):
    return np.stack([-np.sin(lat) * np.cos(lon), -np.sin(lat) * np.sin(lon),
                     np.cos(lat)], 1)


def _cell_centres(ops):
    return np.stack([ops.n_x, ops.n_y, ops.n_z], 1)


def _stack(u, h):
    return np.concatenate([u[:, 0], u[:, 1], u[:, 2], h])


def _harmonic_noise(rng, lat, lon, lmax=8, rms=10.0):
    theta = 0.5 * np.pi - lat
    phi = np.mod(lon, 2.0 * np.pi)
    field = np.zeros_like(lat)
    for ell in range(1, lmax + 1):
        for m in range(0, ell + 1):
            y = sph_harm_y(ell, m, theta, phi)
            field += rng.standard_normal() * y.real
            if m > 0:
                field += rng.standard_normal() * y.imag
    return field * (rms / np.sqrt(np.mean(field * field)))


def balanced_zonal(ops, seed, mean_depth=5960.0, radius=EARTH_RADIUS,
                   omega=EARTH_OMEGA, g=GRAVITY):
    """C0 construction: u = u0 cos(lat) zonal, u0 ~ U(20,40), balanced h
    (g h = g h0 - (a Omega u0 + u0^2/2) sin^2 lat) plus an rms-10 m
    harmonic perturbation of degree <= 8."""
    rng = np.random.default_rng(seed)
    x = _cell_centres(ops)
    lat, lon = _latlon(x)
    u0 = rng.uniform(20.0, 40.0)
    u = (u0 * np.cos(lat))[:, None] * _zonal_unit(lon)
    k = (radius * omega * u0 + 0.5 * u0 * u0) / g
    h0 = mean_depth + k / 3.0
    h = h0 - k * np.sin(lat) ** 2
    h = h + _harmonic_noise(rng, lat, lon)
    return _stack(u, h), rng


def config0_state(ops, seed=0):
    return balanced_zonal(ops, seed)[0]


def config1_state(ops, seed=1, zeta_amp=8e-6, radius=EARTH_RADIUS):
    state, _ = balanced_zonal(ops, seed)
    x = _cell_centres(ops)
    lat, lon = _latlon(x)
    # zeta = -30 psi / a^2 for the degree-5 pattern; max of cos^4 sin is
    # 16 / (25 sqrt 5)
    K = zeta_amp / (30.0 * 16.0 / (25.0 * np.sqrt(5.0)))
    c, s = np.cos(lat), np.sin(lat)
    u_lon = radius * K * np.cos(4 * lon) * c ** 3 * (c * c - 4.0 * s * s)
    u_lat = 4.0 * radius * K * c ** 3 * s * np.sin(4 * lon)
    du = u_lon[:, None] * _zonal_unit(lon) + u_lat[:, None] * _merid_unit(lat, lon)
    N = ops.n_g
    for k in range(3):
        state[k * N:(k + 1) * N] += du[:, k]
    return state


def config2_state(ops, seed=3, u0=20.0, peak=2000.0, efold=1.5e6,
                  mean_depth=5960.0, radius=EARTH_RADIUS, omega=EARTH_OMEGA,
                  g=GRAVITY):
    """Returns (state, h_s): zonal u0 cos(lat) over a Gaussian bump."""
    rng = np.random.default_rng(seed)
    x = _cell_centres(ops)
    lat, lon = _latlon(x)
    lat_c = np.deg2rad(rng.uniform(-45.0, 45.0))
    lon_c = np.deg2rad(rng.uniform(0.0, 360.0))
    xc = np.array([np.cos(lat_c) * np.cos(lon_c), np.cos(lat_c) * np.sin(lon_c),
                   np.sin(lat_c)])
    r = radius * np.arccos(np.clip(x @ xc, -1.0, 1.0))
    h_s = peak * np.exp(-(r / efold) ** 2)
    u = (u0 * np.cos(lat))[:, None] * _zonal_unit(lon)
    k = (radius * omega * u0 + 0.5 * u0 * u0) / g
    h0 = mean_depth + k / 3.0
    h = h0 - k * np.sin(lat) ** 2 - h_s
    return _stack(u, h), h_s


def config3_state(ops, seed=4, u_max=60.0, half_width_deg=10.0,
                  mean_depth=10000.0, noise_rms=1.0, radius=EARTH_RADIUS,
                  omega=EARTH_OMEGA, g=GRAVITY):
    """Zonal jet centred at lat0 ~ U(30,55) deg with the balanced height
    (quadrature of g dh/dlat = -a u (f + u tan(lat)/a)) plus white noise."""
    rng = np.random.default_rng(seed)
    lat0 = np.deg2rad(rng.uniform(30.0, 55.0))
    w = np.deg2rad(half_width_deg)

    def jet(phi):
        return u_max * np.exp(-((phi - lat0) / w) ** 2)

    phi = np.linspace(-0.5 * np.pi, 0.5 * np.pi, 40001)
    uj = jet(phi)
    dh = -(radius / g) * uj * (2.0 * omega * np.sin(phi)
                               + uj * np.tan(np.clip(phi, -1.5707, 1.5707)) / radius)
    hprof = np.concatenate([[0.0], np.cumsum(0.5 * (dh[1:] + dh[:-1]) * np.diff(phi))])
    # area-weighted mean of the profile over the sphere
    wts = np.cos(phi)
    mean_prof = np.sum(hprof * wts) / np.sum(wts)
    x = _cell_centres(ops)
    lat, lon = _latlon(x)
    h = mean_depth + np.interp(lat, phi, hprof) - mean_prof
    u = jet(lat)[:, None] * _zonal_unit(lon)
    noise = rng.standard_normal(lat.shape[0])
    noise -= noise.mean()
    noise *= noise_rms / np.sqrt(np.mean(noise * noise))
    return _stack(u, h + noise)


def config4_state(ops, seed=2):
    return balanced_zonal(ops, seed)[0]


def make_config(name, level=None):
    """(ops, u0, spec) for a named config; ``level`` overrides the grid."""
    from .grid import cached_sphere_operators
    spec = CONFIGS[name]
    lvl = spec.level if level is None else int(level)
    ops = cached_sphere_operators(lvl)
    if name == "C0":
        u0 = config0_state(ops, spec.seed)
    elif name == "C1":
        u0 = config1_state(ops, spec.seed)
    elif name == "C2":
        u0, h_s = config2_state(ops, spec.seed)
        ops = ops.with_surface(h_s)
    elif name == "C3":
        u0 = config3_state(ops, spec.seed)
    else:
        u0 = config4_state(ops, spec.seed)
    return ops, u0, spec
