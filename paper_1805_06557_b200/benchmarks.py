"""Benchmark initial state and error metric.

* ``init_barotropic_instability`` -- the balanced mid-latitude jet of the
  published barotropic-instability test (Galewsky, Scott & Polvani 2004),
  optionally with the Gaussian height bump; the same construction as the
  reference (benchmarks.py:147-215): the jet is projected on the truncation
  by a device ``vortdiv_from_uv``, the balancing height integrates
  ``u (f + u tan(lat) / a)`` from the south pole with adaptive quadrature of
  the *projected* jet, is recentred to zero global mean, and the height field
  goes back to spectral space with the device analysis.
* ``linf_error`` -- max-abs grid difference (benchmarks.py:290-306), height
  in metres.

The quadrature is host-side by nature (scipy's adaptive ``quad`` calls back
into Python per latitude); the transforms run on the GPU.
"""

from __future__ import annotations

import math

import numpy as np

from .errors import ConfigurationError, DataError
from .sphere import (GridField, SpectralField, SphereConfig, analysis, plan_for, synthesis,
                     vortdiv_from_uv)
from .swe import PrognosticState

# published test-case constants: angles in radians, heights in m, speeds in m/s
GALEWSKY = {
    "u_max": 80.0,
    "jet_lat_south": math.pi / 7.0,
    "jet_lat_north": math.pi / 2.0 - math.pi / 7.0,
    "bump_amplitude": 120.0,
    "bump_half_width_lon": 1.0 / 3.0,
    "bump_half_width_lat": 1.0 / 15.0,
    "bump_center_lat": math.pi / 4.0,
    "mean_height": 10000.0,
}


def load_benchmark_constants() -> dict:
    return dict(GALEWSKY)


def jet_velocity(lat, c=GALEWSKY) -> np.ndarray:
    """u(lat) = u_max / e_n exp(1 / ((lat - lat0)(lat - lat1))) inside the jet, else 0."""
    lat = np.asarray(lat, dtype=float)
    lat0, lat1 = c["jet_lat_south"], c["jet_lat_north"]
    e_n = math.exp(-4.0 / (lat1 - lat0) ** 2)
    out = np.zeros_like(lat)
    inside = (lat > lat0) & (lat < lat1)
    x = lat[inside]
    out[inside] = (c["u_max"] / e_n) * np.exp(1.0 / ((x - lat0) * (x - lat1)))
    return out


def zonal_velocity_evaluator(vort: SpectralField, cfg: SphereConfig):
    """u(lat) of a zonal state from its m = 0 stream function, at any latitude
    (the balance integrand must see the truncation-projected jet):
    u = -(1/a) dpsi/dlat, psi_l = -a^2 vort_l0 / (l (l+1)),
    dPbar_l/dlat = ((l+1) e_l Pbar_{l-1} - l e_{l+1} Pbar_{l+1}) / cos(lat),
    e_l = sqrt(l^2 / (4 l^2 - 1)) (sphere.py:96-111, benchmarks.py:118-140)."""
    trunc = vort.trunc
    l = np.arange(trunc + 2, dtype=float)
    ll1 = l[: trunc + 1] * (l[: trunc + 1] + 1.0)
    psi = np.zeros(trunc + 1)
    psi[1:] = -cfg.radius_a ** 2 * np.real(vort.coeffs[1:, 0]) / ll1[1:]
    with np.errstate(divide="ignore", invalid="ignore"):
        e = np.sqrt(l * l / (4.0 * l * l - 1.0))
    e[0] = 0.0

    def u_at(lat: float) -> float:
        x, cos = math.sin(lat), math.cos(lat)
        p = np.empty(trunc + 2)
        p[0] = 1.0 / math.sqrt(4.0 * math.pi)
        p[1] = math.sqrt(3.0) * x * p[0]
        for k in range(2, trunc + 2):
            p[k] = (x * p[k - 1] - e[k - 1] * p[k - 2]) / e[k]
        k = np.arange(1, trunc + 1)
        dp = ((k + 1) * e[k] * p[k - 1] - k * e[k + 1] * p[k + 1]) / cos
        return float(-np.dot(psi[1:], dp) / cfg.radius_a)

    return u_at


def init_barotropic_instability(cfg: SphereConfig, with_bump: bool = True,
                                constants: dict | None = None) -> PrognosticState:
    """Balanced zonal jet (+ height bump): benchmarks.py:147-215."""
    from scipy.integrate import quad

    c = dict(GALEWSKY if constants is None else constants)
    plan = plan_for(cfg)
    a, g = cfg.radius_a, cfg.gravity_g
    u_grid = np.repeat(jet_velocity(plan.lats, c)[:, None], cfg.nlon, axis=1)
    vort, _ = vortdiv_from_uv(GridField(u_grid, cfg), GridField(np.zeros_like(u_grid), cfg), cfg)
    vort.coeffs[:, 1:] = 0.0  # exactly zonal
    div = SpectralField.zeros(cfg.trunc)
    u_t = zonal_velocity_evaluator(vort, cfg)

    def integrand(lat):
        u = u_t(lat)
        return a * u * (2.0 * cfg.omega * math.sin(lat) + math.tan(lat) * u / a)

    lat0, lat1 = c["jet_lat_south"], c["jet_lat_north"]
    gh = np.empty(cfg.nlat)
    for j, lat in enumerate(plan.lats):
        val, _ = quad(integrand, -math.pi / 2, lat,
                      points=[q for q in (lat0, lat1) if -math.pi / 2 < q < lat],
                      limit=200, epsabs=1e-12, epsrel=1e-12)
        if not np.isfinite(val):
            raise DataError("balance integral failed to converge")
        gh[j] = -val
    gh -= np.sum(plan.weights * gh) / 2.0  # zero global mean
    phi_grid = np.repeat(gh[:, None], cfg.nlon, axis=1)
    if with_bump:
        lon = plan.lons[None, :]
        lat = plan.lats[:, None]
        lon_c = np.where(lon > math.pi, lon - 2.0 * math.pi, lon)  # bump centred at lon 0
        shape = (np.cos(lat) * np.exp(-((lon_c / c["bump_half_width_lon"]) ** 2))
                 * np.exp(-(((c["bump_center_lat"] - lat) / c["bump_half_width_lat"]) ** 2)))
        phi_grid = phi_grid + g * c["bump_amplitude"] * shape
    phi = analysis(GridField(phi_grid, cfg), cfg)
    return PrognosticState(phi, vort, div, cfg)


def linf_error(state: PrognosticState, reference: PrognosticState, field: str = "h") -> float:
    """Max-abs grid difference of one field; "h" is the height in metres."""
    if state.cfg != reference.cfg:
        raise ConfigurationError("state and reference use different grids")
    pick = {"h": "phi_pert", "vort": "vort", "div": "div"}
    if field not in pick:
        raise ConfigurationError(f"unknown error field {field!r}")
    cfg = state.cfg
    x = synthesis(getattr(state, pick[field]), cfg).values
    y = synthesis(getattr(reference, pick[field]), cfg).values
    if field == "h":
        x, y = x / cfg.gravity_g, y / cfg.gravity_g
    return float(np.max(np.abs(x - y)))
