"""Sphere grid, plans and spectral transforms (host mirror of swerexi.sphere).

API-compatible with /root/reference/pkg/src/swerexi/sphere.py for
real-origin fields: ``SphereConfig`` (115-160), ``SpectralField`` (235-262),
``GridField`` (265-270), ``gauss_legendre_nodes`` (31-58), ``plan_for``
(231-232), ``analysis`` (297-315), ``synthesis`` (318-339), ``laplacian``
(350-355), ``inv_laplacian`` (358-366), ``uv_from_vortdiv`` (375-402).
Transforms execute on the GPU through libswx (``swx_sht_*``); the grid
nodes and sectoral seeds are computed here once per plan.
Complex-origin fields (``neg_coeffs``) are outside the B200 hot path and
raise ``ConfigurationError``.
"""

from __future__ import annotations

import ctypes
import dataclasses
import functools
import math

import numpy as np

from . import _lib
from .device import ncoef, pack, ptr, stream_ptr, to_device, unpack
from .errors import ConfigurationError, DataError

EARTH_RADIUS = 6.37122e6
EARTH_OMEGA = 7.292e-5
EARTH_GRAVITY = 9.80616


def gauss_legendre_nodes(n: int) -> tuple[np.ndarray, np.ndarray]:
    """Gauss-Legendre nodes (ascending) and weights by Newton iteration on
    P_n from the cosine guess -- the reference's node recipe
    (sphere.py:31-58), so plans agree with it to the last bits."""
    if n < 1:
        raise ConfigurationError(f"need at least one latitude node, got {n}")
    x = np.cos(np.pi * (np.arange(n) + 0.75) / (n + 0.5))

    def pn_and_prev(x):
        prev, cur = np.zeros_like(x), np.ones_like(x)
        for d in range(1, n + 1):
            prev, cur = cur, ((2 * d - 1) * x * cur - (d - 1) * prev) / d
        return cur, prev

    for _ in range(100):
        pn, pm = pn_and_prev(x)
        dx = pn / (n * (x * pn - pm) / (x * x - 1.0))
        x = x - dx
        if np.max(np.abs(dx)) < 1e-15:
            break
    pn, pm = pn_and_prev(x)
    deriv = n * (x * pn - pm) / (x * x - 1.0)
    w = 2.0 / ((1.0 - x * x) * deriv * deriv)
    order = np.argsort(x)
    return x[order], w[order]


def sectoral_seeds(trunc: int, x: np.ndarray) -> np.ndarray:
    """Pbar_m^m(x_j) as a (T+1, nlat) table, accumulated in mantissa/exponent
    form so it cannot underflow before reconstitution (sphere.py:86-95)."""
    cosl = np.sqrt(1.0 - x * x)
    out = np.empty((trunc + 1, x.size))
    mant = np.full(x.size, 1.0 / math.sqrt(4.0 * math.pi))
    expo = np.zeros(x.size, dtype=np.int64)
    out[0] = np.ldexp(mant, expo)
    for m in range(1, trunc + 1):
        mant, e = np.frexp(mant * (math.sqrt((2 * m + 1) / (2.0 * m)) * cosl))
        expo += e
        out[m] = np.ldexp(mant, expo)
    return out


@dataclasses.dataclass(frozen=True)
class SphereConfig:
    """Grid and planetary constants for one triangular truncation."""

    trunc: int
    nlat: int
    nlon: int
    radius_a: float = EARTH_RADIUS
    omega: float = EARTH_OMEGA
    gravity_g: float = EARTH_GRAVITY

    def __post_init__(self):
        if self.trunc < 0:
            raise ConfigurationError(f"truncation must be >= 0, got {self.trunc}")
        if self.nlat < self.trunc + 1:
            raise ConfigurationError(
                f"nlat={self.nlat} too small for T{self.trunc} (need >= {self.trunc + 1})")
        need = math.ceil((3 * self.trunc + 1) / 2)
        if self.nlat < need:
            raise ConfigurationError(
                f"nlat={self.nlat} violates 3/2-rule dealiasing for T{self.trunc} (need >= {need})")
        if self.nlon < 2 * self.nlat:
            raise ConfigurationError(f"nlon={self.nlon} must be at least 2*nlat={2 * self.nlat}")
        if self.radius_a <= 0 or self.gravity_g <= 0:
            raise ConfigurationError("radius and gravity must be positive")
        if self.omega < 0:
            raise ConfigurationError("rotation rate must be >= 0")

    @classmethod
    def for_truncation(cls, trunc: int, radius_a: float = EARTH_RADIUS,
                       omega: float = EARTH_OMEGA, gravity_g: float = EARTH_GRAVITY):
        """Smallest even dealiased grid (T42 -> 64 x 128, T256 -> 386 x 772)."""
        nlat = math.ceil((3 * trunc + 1) / 2)
        nlat += nlat % 2
        return cls(trunc, nlat, 2 * nlat, radius_a, omega, gravity_g)


@dataclasses.dataclass
class SpectralField:
    """Triangular-truncated SH coefficients ``coeffs[l, m]`` (m <= l)."""

    coeffs: np.ndarray
    neg_coeffs: np.ndarray | None = None

    @property
    def trunc(self) -> int:
        return self.coeffs.shape[0] - 1

    @property
    def value_kind(self) -> str:
        return "real-origin" if self.neg_coeffs is None else "complex-origin"

    def copy(self) -> "SpectralField":
        return SpectralField(self.coeffs.copy(),
                             None if self.neg_coeffs is None else self.neg_coeffs.copy())

    @classmethod
    def zeros(cls, trunc: int) -> "SpectralField":
        return cls(np.zeros((trunc + 1, trunc + 1), dtype=np.complex128))


@dataclasses.dataclass
class GridField:
    """Values on the Gauss-Legendre x equiangular grid."""

    values: np.ndarray
    grid: SphereConfig


class ShtPlan:
    """Device transform plan (the SpherePlan analogue, sphere.py:163-223).

    Owns the libswx plan, a reusable workspace and the host-side grid
    description; thread-confined to the device it was created on.
    """

    def __init__(self, cfg: SphereConfig):
        import torch

        self.cfg = cfg
        lib = _lib.lib()
        x, w = gauss_legendre_nodes(cfg.nlat)
        self.sin_lat, self.weights = x, w
        self.cos_lat = np.sqrt(1.0 - x * x)
        self.lats = np.arcsin(x)
        self.lons = 2.0 * np.pi * np.arange(cfg.nlon) / cfg.nlon
        l = np.arange(cfg.trunc + 1)
        self.ll1 = (l * (l + 1)).astype(float)
        seeds = np.ascontiguousarray(sectoral_seeds(cfg.trunc, x))
        h = ctypes.c_void_p()
        _lib.check(lib.swx_sht_create(
            ctypes.byref(h), cfg.trunc, cfg.nlat, cfg.nlon, cfg.radius_a, cfg.omega,
            x.ctypes.data, w.ctypes.data, seeds.ctypes.data))
        self._h = h
        self._lib = lib
        self.device = torch.device("cuda", torch.cuda.current_device())
        nbytes = lib.swx_sht_workspace_bytes(h)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.swx_sht_destroy(h)
            except Exception:
                pass

    # device-level entry points (tensors in, tensors out) -------------------
    def synthesis_dev(self, coeffs, out=None, stream=None):
        """(nf, ncoef) complex128 -> (nf, nlat, nlon) float64."""
        import torch

        nf = coeffs.shape[0]
        if out is None:
            out = torch.empty((nf, self.cfg.nlat, self.cfg.nlon), dtype=torch.float64,
                              device=self.device)
        _lib.check(self._lib.swx_sht_synthesis(
            self._h, nf, ptr(coeffs), ptr(out), ptr(self.workspace), self.workspace.numel(),
            stream_ptr(stream)))
        return out

    def analysis_dev(self, grids, out=None, stream=None):
        import torch

        nf = grids.shape[0]
        if out is None:
            out = torch.empty((nf, ncoef(self.cfg.trunc)), dtype=torch.complex128,
                              device=self.device)
        _lib.check(self._lib.swx_sht_analysis(
            self._h, nf, ptr(grids), ptr(out), ptr(self.workspace), self.workspace.numel(),
            stream_ptr(stream)))
        return out

    def uv_dev(self, vort, div, stream=None):
        import torch

        shape = (self.cfg.nlat, self.cfg.nlon)
        u = torch.empty(shape, dtype=torch.float64, device=self.device)
        v = torch.empty(shape, dtype=torch.float64, device=self.device)
        _lib.check(self._lib.swx_sht_uv(
            self._h, ptr(vort), ptr(div), ptr(u), ptr(v), ptr(self.workspace),
            self.workspace.numel(), stream_ptr(stream)))
        return u, v

    def vortdiv_dev(self, u, v, stream=None):
        import torch

        vort = torch.empty(ncoef(self.cfg.trunc), dtype=torch.complex128, device=self.device)
        div = torch.empty_like(vort)
        _lib.check(self._lib.swx_sht_vortdiv(
            self._h, ptr(u), ptr(v), ptr(vort), ptr(div), ptr(self.workspace),
            self.workspace.numel(), stream_ptr(stream)))
        return vort, div

    def set_synth_event(self, event=None):
        """Record ``event`` (torch.cuda.Event) after the synthesis of each
        following tendency call (None clears)."""
        _lib.check(self._lib.swx_sht_set_synth_event(
            self._h, event.cuda_event if event is not None else 0))

    def set_done_signal(self, on: bool) -> int:
        """While on, the following tendency calls count each completed table-
        analysis item in per-column device counters (and bump a generation
        counter per call), whose address is returned (0 if the plan has no
        table analysis): an lg pole sum given that address (``ready=``) right
        after a signalled tendency on the same stream starts on columns as they
        complete.  The counters only grow, so a signalled call without a
        waiting pole sum is harmless; one stream per plan."""
        if on and not self.fused_stages():
            return 0
        out = ctypes.c_void_p()
        _lib.check(self._lib.swx_sht_set_done_signal(self._h, 1 if on else 0, ctypes.byref(out)))
        return int(out.value or 0)

    def fused_stages(self) -> bool:
        """Whether the tendency has separable stages (fused grid / table path)."""
        return bool(self._lib.swx_sht_has_stages(self._h))

    def tendency_part(self, stage: int, atoms: int, m0: int, m1: int, state=None, out=None,
                      sub=None, stream=None, workspace=None):
        """One stage of the tendency on columns [m0, m1) (swx_sht_tendency_part);
        ``workspace`` (default: the plan's) carries the stage results between
        calls."""
        ws = self.workspace if workspace is None else workspace
        _lib.check(self._lib.swx_sht_tendency_part(
            self._h, int(stage), int(atoms), int(m0), int(m1),
            ptr(state) if state is not None else 0, ptr(sub) if sub is not None else 0,
            ptr(out) if out is not None else 0, ptr(ws), ws.numel(), stream_ptr(stream)))
        return out

    def tendency_dev(self, atoms: int, state, out=None, stream=None, sub=None):
        """out = tendency(state) (minus ``sub`` when given, fused on the device)."""
        import torch

        if out is None:
            out = torch.empty_like(state)
        if sub is None:
            _lib.check(self._lib.swx_sht_tendency(
                self._h, atoms, ptr(state), ptr(out), ptr(self.workspace),
                self.workspace.numel(), stream_ptr(stream)))
        else:
            _lib.check(self._lib.swx_sht_tendency_sub(
                self._h, atoms, ptr(state), ptr(sub), ptr(out), ptr(self.workspace),
                self.workspace.numel(), stream_ptr(stream)))
        return out


@functools.lru_cache(maxsize=8)
def _plan(cfg: SphereConfig) -> ShtPlan:
    return ShtPlan(cfg)


def plan_for(cfg: SphereConfig) -> ShtPlan:
    return _plan(cfg)


def _tri_mask(trunc: int) -> np.ndarray:
    l = np.arange(trunc + 1)[:, None]
    m = np.arange(trunc + 1)[None, :]
    return m <= l


def _check_grid(field: GridField, cfg: SphereConfig):
    if field.values.shape != (cfg.nlat, cfg.nlon):
        raise ConfigurationError(
            f"grid shape {field.values.shape} does not match ({cfg.nlat}, {cfg.nlon})")
    if not np.all(np.isfinite(field.values)):
        raise DataError("grid field contains non-finite values")


def _pad_coeffs(coeffs: np.ndarray, trunc: int) -> np.ndarray:
    n = coeffs.shape[0]
    if n == trunc + 1:
        return coeffs
    out = np.zeros((trunc + 1, trunc + 1), dtype=np.complex128)
    out[:n, :n] = coeffs
    return out


def _require_real_origin(*fields: SpectralField):
    for f in fields:
        if f.neg_coeffs is not None:
            raise ConfigurationError("the B200 transforms take real-origin fields only")


def analysis(grid: GridField, cfg: SphereConfig) -> SpectralField:
    """Forward transform of a real grid (sphere.py:297-315)."""
    import torch

    _check_grid(grid, cfg)
    if np.iscomplexobj(grid.values):
        raise ConfigurationError("complex-valued grids are outside the B200 hot path")
    plan = plan_for(cfg)
    g = torch.from_numpy(np.ascontiguousarray(grid.values, dtype=np.float64)).to(plan.device)
    c = plan.analysis_dev(g[None])
    return SpectralField(unpack(c.cpu().numpy(), cfg.trunc)[0])


def synthesis(spec: SpectralField, cfg: SphereConfig) -> GridField:
    """Inverse transform of a real-origin field (sphere.py:318-339)."""
    if spec.trunc > cfg.trunc:
        raise ConfigurationError(
            f"field truncation T{spec.trunc} exceeds grid truncation T{cfg.trunc}")
    _require_real_origin(spec)
    plan = plan_for(cfg)
    c = to_device(pack(_pad_coeffs(spec.coeffs, cfg.trunc)[None]), plan.device)
    return GridField(plan.synthesis_dev(c)[0].cpu().numpy(), cfg)


def laplacian(spec: SpectralField, cfg: SphereConfig) -> SpectralField:
    """Multiply each (l, m) coefficient by -l(l+1)/a^2 (sphere.py:350-355)."""
    l = np.arange(spec.trunc + 1)
    eig = (-(l * (l + 1)).astype(float) / cfg.radius_a**2)[:, None]
    neg = None if spec.neg_coeffs is None else spec.neg_coeffs * eig
    return SpectralField(spec.coeffs * eig, neg)


def inv_laplacian(spec: SpectralField, cfg: SphereConfig) -> SpectralField:
    """Inverse Laplacian, (0,0) gauge mode -> 0 (sphere.py:358-366)."""
    n = spec.trunc + 1
    l = np.arange(n)
    inv = np.zeros(n)
    inv[1:] = -(cfg.radius_a**2) / (l[1:] * (l[1:] + 1)).astype(float)
    neg = None if spec.neg_coeffs is None else spec.neg_coeffs * inv[:, None]
    return SpectralField(spec.coeffs * inv[:, None], neg)


def uv_from_vortdiv(zeta: SpectralField, delta: SpectralField, cfg: SphereConfig):
    """Grid velocities from vorticity/divergence (sphere.py:375-402)."""
    _require_real_origin(zeta, delta)
    if zeta.trunc != delta.trunc:
        raise ConfigurationError("vorticity/divergence truncations differ")
    plan = plan_for(cfg)
    z = to_device(pack(_pad_coeffs(zeta.coeffs, cfg.trunc)), plan.device)
    d = to_device(pack(_pad_coeffs(delta.coeffs, cfg.trunc)), plan.device)
    u, v = plan.uv_dev(z, d)
    return GridField(u.cpu().numpy(), cfg), GridField(v.cpu().numpy(), cfg)


def vortdiv_from_uv(u: GridField, v: GridField, cfg: SphereConfig):
    """Vorticity and divergence coefficients from grid velocities
    (sphere.py:405-430): one device FFT + table analysis (swx_sht_vortdiv)."""
    _check_grid(u, cfg)
    _check_grid(v, cfg)
    plan = plan_for(cfg)
    import torch

    ug = torch.from_numpy(np.ascontiguousarray(np.real(u.values), dtype=np.float64)).to(plan.device)
    vg = torch.from_numpy(np.ascontiguousarray(np.real(v.values), dtype=np.float64)).to(plan.device)
    z, d = plan.vortdiv_dev(ug, vg)
    return (SpectralField(unpack(z.cpu().numpy(), cfg.trunc)),
            SpectralField(unpack(d.cpu().numpy(), cfg.trunc)))

