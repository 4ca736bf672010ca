"""Oracle: REXI coefficients, linear REXI step, ETD2RK step, seeded inputs.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
(/root/reference/pkg/src/swerexi/):

  * ``phi_function``                         rexi.py:74-98
  * ``shifted_contour_from_points``          rexi.py:101-115
  * ``circle_contour_coeffs``                rexi.py:140-167
  * ``rexi_step``                            steppers.py:214-235
  * ``etdrk2_generic`` / ``etdrk2_step``     steppers.py:238-269
  * ``_state_blown_up``                      steppers.py:516-520
and the seeded synthetic inputs of SURVEY §8(d).
"""

from __future__ import annotations

import math

import numpy as np

from . import rexi as orx
from . import sht as osh


# ----------------------------------------------------------------------
# coefficients

def psi(k: int, z):
    z = np.asarray(z, dtype=np.complex128)
    if k == 0:
        return np.exp(z)
    small = np.abs(z) < 1e-2
    zs = np.where(small, 1.0, z)
    with np.errstate(over="ignore", invalid="ignore"):
        if k == 1:
            out = (np.exp(zs) - 1.0) / zs
        else:
            out = (np.exp(zs) - 1.0 - zs) / (zs * zs)
    if small.any():
        acc = np.zeros_like(z)
        for j in range(7, -1, -1):
            acc = acc * z + 1.0 / math.factorial(j + k)
        out = np.where(small, acc, out)
    return out


def contour_coeffs(k: int, p0: float = 10.0, p1: float = 30.0, n: int = 128):
    """(alphas, betas) on the circle through p0 and +-i p1."""
    r = (p0 * p0 + p1 * p1) / (2.0 * p0)
    center = complex(p0 - r)
    theta = 2.0 * np.pi * np.arange(1, n + 1) / n
    ring = r * np.exp(1j * theta)
    z = ring + center
    f = psi(k, z)
    return -z, -(ring / n) * f


# ----------------------------------------------------------------------
# steps on dense (3, n, n) stacks

def rexi_step(group, model: orx.Model, dt, alphas, betas, stack, factors=None):
    return orx.rexi_sum(group, model, dt, alphas, betas, stack, factors)


def etdrk2_step(model: orx.Model, grid: osh.Grid, dt: float, coeff_sets, stack,
                group: str = "lg", remainder: str = "lc_n", factors=None):
    """ETD2RK with ``group`` (lg | l) by REXI and ``remainder`` (lc_n | n) as the
    non-linear part (steppers.py:238-269; tendency_group swe.py:254-279).

    ``coeff_sets[k] = (alphas, betas_k)`` for psi_k, k = 0, 1, 2.
    """
    def apply_psi(k, v):
        a, b = coeff_sets[k]
        return orx.rexi_sum(group, model, dt, a, b, v, factors)

    rhs = grid.tendency_lc_n if remainder == "lc_n" else grid.tendency_n
    nu = rhs(stack)
    a = apply_psi(0, stack) + apply_psi(1, nu) * dt
    na = rhs(a)
    return a + apply_psi(2, na - nu) * dt


def blown_up(grid: osh.Grid, stack) -> bool:
    if not np.all(np.isfinite(stack)):
        return True
    return bool(np.max(np.abs(grid.synthesis(stack[0]))) > 1.0e6)


# ----------------------------------------------------------------------
# seeded synthetic inputs

def seeded_linear_state(trunc: int, seed: int = 0) -> np.ndarray:
    """cfg0/1/4 input: amplitudes 1e3, 1e-5, 1e-5 with (l+1)^-2 decay."""
    rng = np.random.default_rng(seed)
    n = trunc + 1
    l = np.arange(n)[:, None]
    m = np.arange(n)[None, :]
    out = np.zeros((3, n, n), dtype=np.complex128)
    for f, amp in enumerate((1e3, 1e-5, 1e-5)):
        c = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * amp / (l + 1.0) ** 2
        c[m > l] = 0.0
        c[:, 0] = c[:, 0].real
        out[f] = c
    return out


def seeded_balanced_state(grid: osh.Grid, peak: float = 1e-5, seed: int = 0) -> np.ndarray:
    """cfg2/3 input: random vorticity ~ (l+1)^-1.5 scaled to max|zeta| = peak,
    zero divergence, linearly balanced phi'."""
    trunc = grid.trunc
    rng = np.random.default_rng(seed)
    n = trunc + 1
    l = np.arange(n)[:, None]
    m = np.arange(n)[None, :]
    c = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / (l + 1.0) ** 1.5
    c[m > l] = 0.0
    c[:, 0] = c[:, 0].real
    c[0, 0] = 0.0
    zmax = np.max(np.abs(grid.synthesis(c)))
    c = c * (peak / zmax)
    st = np.zeros((3, n, n), dtype=np.complex128)
    st[1] = c
    lc = grid.tendency_lc(st)
    kap = grid.ll1 / grid.radius**2
    phi = np.zeros((n, n), dtype=np.complex128)
    phi[1:] = -lc[2][1:] / kap[1:, None]
    st[0] = phi
    return st
