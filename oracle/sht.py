"""Oracle: Gauss grid, Legendre tables, SH transforms, SWE tendencies.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
(/root/reference/pkg/src/swerexi/):

  * ``gauss_legendre_nodes``                sphere.py:31-58
  * ``_legendre_tables`` (P and H=dP/dlat)  sphere.py:72-112
  * ``SphereConfig.for_truncation``         sphere.py:148-160
  * ``analysis`` / ``synthesis``            sphere.py:297-347 (+212-223)
  * ``laplacian`` / ``inv_laplacian``       sphere.py:350-366
  * ``uv_from_vortdiv`` / ``vortdiv_from_uv`` sphere.py:375-430
  * ``tendency_lc`` / ``tendency_n`` / group LC_N   swe.py:188-279

Normalisation: orthonormal, no Condon-Shortley phase (sphere.py:3-13).
"""

from __future__ import annotations

import functools
import math

import numpy as np

G_EARTH = 9.80616          # sphere.py:28


def grid_for_truncation(trunc: int) -> tuple[int, int]:
    """Smallest even 3/2-dealiased grid (sphere.py:148-160)."""
    nlat = math.ceil((3 * trunc + 1) / 2)
    nlat += nlat % 2
    return nlat, 2 * nlat


def gauss_nodes(n: int) -> tuple[np.ndarray, np.ndarray]:
    """Newton on P_n from cos(pi(k+3/4)/(n+1/2)); ascending (sphere.py:31-58)."""
    x = np.cos(np.pi * (np.arange(n) + 0.75) / (n + 0.5))

    def legendre_pair(x):
        p0, p1 = np.zeros_like(x), np.ones_like(x)
        for d in range(1, n + 1):
            p0, p1 = p1, ((2 * d - 1) * x * p1 - (d - 1) * p0) / d
        return p1, n * (x * p1 - p0) / (x * x - 1.0)

    for _ in range(100):
        p, dp = legendre_pair(x)
        step = p / dp
        x = x - step
        if np.max(np.abs(step)) < 1e-15:
            break
    _, dp = legendre_pair(x)
    w = 2.0 / ((1.0 - x * x) * dp * dp)
    o = np.argsort(x)
    return x[o], w[o]


def legendre_tables(trunc: int, x: np.ndarray):
    """P[j, l, m] (l <= T+1) and H[j, l, m] = dP/dlat (l <= T) with the
    mantissa/exponent sectoral seed (sphere.py:72-112)."""
    nj = x.size
    cosl = np.sqrt(1.0 - x * x)
    L = trunc + 1
    P = np.zeros((nj, L + 1, trunc + 1))
    mant = np.full(nj, 1.0 / math.sqrt(4.0 * math.pi))
    expo = np.zeros(nj, dtype=np.int64)
    for m in range(trunc + 1):
        if m:
            mant, e = np.frexp(mant * (math.sqrt((2 * m + 1) / (2.0 * m)) * cosl))
            expo += e
        seed = np.ldexp(mant, expo)
        P[:, m, m] = seed
        if m + 1 <= L:
            P[:, m + 1, m] = math.sqrt(2 * m + 3) * x * seed
        for l in range(m + 2, L + 1):
            e1 = math.sqrt((l * l - m * m) / (4.0 * l * l - 1.0))
            e0 = math.sqrt(((l - 1) ** 2 - m * m) / (4.0 * (l - 1) ** 2 - 1.0))
            P[:, l, m] = (x * P[:, l - 1, m] - e0 * P[:, l - 2, m]) / e1
    H = np.zeros((nj, trunc + 1, trunc + 1))
    for m in range(trunc + 1):
        ls = np.arange(m, trunc + 1).astype(float)
        el = _eps(ls, m)
        elp = _eps(ls + 1, m)
        below = np.zeros((nj, ls.size))
        below[:, 1:] = P[:, m:trunc, m]
        above = P[:, m + 1:trunc + 2, m]
        H[:, m:, m] = ((ls + 1) * el * below - ls * elp * above) / cosl[:, None]
    return P, H


def _eps(l, m):
    l = np.asarray(l, dtype=float)
    num = l * l - m * m
    out = np.zeros_like(l)
    ok = num > 0
    out[ok] = np.sqrt(num[ok] / (4.0 * l[ok] * l[ok] - 1.0))
    return out


class Grid:
    """Transform plan for one (T, nlat, nlon) (sphere.py:163-223)."""

    def __init__(self, trunc: int, nlat: int | None = None, nlon: int | None = None,
                 radius: float = 6.37122e6, omega: float = 7.292e-5):
        if nlat is None:
            nlat, nlon = grid_for_truncation(trunc)
        self.trunc, self.nlat, self.nlon = trunc, nlat, nlon
        self.radius, self.omega = radius, omega
        x, w = gauss_nodes(nlat)
        P, H = legendre_tables(trunc, x)
        self.sinl, self.w = x, w
        self.cosl = np.sqrt(1.0 - x * x)
        self.P = np.ascontiguousarray(P[:, : trunc + 1, :])
        self.H = H
        self.dlon = 2.0 * np.pi / nlon
        self.ms = np.arange(trunc + 1)
        self.ll1 = (self.ms * (self.ms + 1)).astype(float)
        # per-m contraction operands, (m, l, j) and (m, j, l)
        self.tabs = {"p": self.P, "h": self.H}
        self._mlj = {k: np.ascontiguousarray(v.transpose(2, 1, 0)) for k, v in self.tabs.items()}
        self._mjl = {k: np.ascontiguousarray(v.transpose(2, 0, 1)) for k, v in self.tabs.items()}

    # Legendre contractions ------------------------------------------
    def legendre_analysis(self, four: np.ndarray, table: str, wts: np.ndarray) -> np.ndarray:
        """c[l, m] = sum_j wts_j table[j,l,m] four[j,m]  (sphere.py:212-217)."""
        fw = four * wts[:, None]
        ri = np.stack([fw.real.T, fw.imag.T], axis=2)
        res = self._mlj[table] @ ri
        return np.ascontiguousarray((res[..., 0] + 1j * res[..., 1]).T)

    def legendre_synthesis(self, coeffs: np.ndarray, table: str) -> np.ndarray:
        """G[j, m] = sum_l table[j,l,m] coeffs[l,m]  (sphere.py:219-223)."""
        ri = np.stack([coeffs.real.T, coeffs.imag.T], axis=2)
        res = self._mjl[table] @ ri
        return np.ascontiguousarray((res[..., 0] + 1j * res[..., 1]).T)

    # full transforms (real-origin fields) ----------------------------
    def to_grid_from_fourier(self, g: np.ndarray) -> np.ndarray:
        """Real grid from m>=0 Fourier columns (sphere.py:342-347)."""
        half = np.zeros((self.nlat, self.nlon // 2 + 1), dtype=np.complex128)
        half[:, : g.shape[1]] = g
        return np.fft.irfft(half, n=self.nlon, axis=1) * self.nlon

    def synthesis(self, coeffs: np.ndarray) -> np.ndarray:
        """sphere.py:318-339 (real-origin branch)."""
        return self.to_grid_from_fourier(self.legendre_synthesis(coeffs, "p"))

    def fourier(self, grid: np.ndarray) -> np.ndarray:
        return np.fft.fft(grid, axis=1)[:, : self.trunc + 1] * self.dlon

    def analysis(self, grid: np.ndarray) -> np.ndarray:
        """sphere.py:297-315 (real grid branch)."""
        f = np.fft.fft(grid, axis=1) * self.dlon
        return self.legendre_analysis(f[:, : self.trunc + 1], "p", self.w)

    # spectral operators -----------------------------------------------
    def laplacian(self, c):
        return c * (-self.ll1 / self.radius**2)[:, None]

    def inv_laplacian(self, c):
        inv = np.zeros(self.trunc + 1)
        inv[1:] = -(self.radius**2) / self.ll1[1:]
        return c * inv[:, None]

    def uv_from_vortdiv(self, vort, div):
        """sphere.py:375-402."""
        a = self.radius
        psi = self.inv_laplacian(vort)
        chi = self.inv_laplacian(div)
        im = 1j * self.ms[None, :]
        g = self.to_grid_from_fourier
        dpsi_lat = g(self.legendre_synthesis(psi, "h"))
        dchi_lat = g(self.legendre_synthesis(chi, "h"))
        dpsi_lon = g(self.legendre_synthesis(psi * im, "p"))
        dchi_lon = g(self.legendre_synthesis(chi * im, "p"))
        sec = 1.0 / self.cosl[:, None]
        return (dchi_lon * sec - dpsi_lat) / a, (dpsi_lon * sec + dchi_lat) / a

    def vortdiv_from_uv(self, u, v):
        """sphere.py:405-430."""
        a = self.radius
        fu, fv = self.fourier(u), self.fourier(v)
        im = 1j * self.ms[None, :]
        woc = self.w / self.cosl
        iq_u = self.legendre_analysis(fu, "p", woc)
        iq_v = self.legendre_analysis(fv, "p", woc)
        ih_u = self.legendre_analysis(fu, "h", self.w)
        ih_v = self.legendre_analysis(fv, "h", self.w)
        return (im * iq_v + ih_u) / a, (im * iq_u - ih_v) / a

    # tendencies ---------------------------------------------------------
    def tendency_lc(self, stack, uv=None):
        """swe.py:188-211."""
        z = np.zeros_like(stack[0])
        if self.omega == 0.0:
            return np.stack([z, z, z])
        if uv is None:
            uv = self.uv_from_vortdiv(stack[1], stack[2])
        u, v = uv
        f = 2.0 * self.omega * self.sinl[:, None]
        fp = 2.0 * self.omega * self.cosl[:, None] / self.radius
        vg = self.synthesis(stack[1])
        dg = self.synthesis(stack[2])
        dvort = self.analysis(-f * dg - fp * v)
        ddiv = self.analysis(f * vg - fp * u)
        return np.stack([z, dvort, ddiv])

    def tendency_n(self, stack, uv=None):
        """swe.py:214-251."""
        if uv is None:
            uv = self.uv_from_vortdiv(stack[1], stack[2])
        u, v = uv
        pg = self.synthesis(stack[0])
        vg = self.synthesis(stack[1])
        _, div_pf = self.vortdiv_from_uv(pg * u, pg * v)
        curl_zf, div_zf = self.vortdiv_from_uv(vg * u, vg * v)
        ke = self.analysis(0.5 * (u**2 + v**2))
        return np.stack([-div_pf, -div_zf, curl_zf - self.laplacian(ke)])

    def tendency_lg(self, stack, phibar):
        """swe.py:169-185."""
        kap = (self.ll1 / self.radius**2)[:, None]
        return np.stack([-phibar * stack[2], np.zeros_like(stack[1]), kap * stack[0]])

    def tendency_lc_n(self, stack):
        """tendency_group(LC_N): lc + n with the shared uv (swe.py:254-279)."""
        uv = self.uv_from_vortdiv(stack[1], stack[2])
        return self.tendency_lc(stack, uv) + self.tendency_n(stack, uv)


@functools.lru_cache(maxsize=8)
def grid_for(trunc: int, nlat: int | None = None, nlon: int | None = None,
             radius: float = 6.37122e6, omega: float = 7.292e-5) -> Grid:
    return Grid(trunc, nlat, nlon, radius, omega)
