"""Oracle: shifted solves, REXI pole sum, tree reduction, realify.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates

  * the gravity ("lg") closed-form 2x2 solve       solvers.py:86-108
  * the Coriolis ("l") band assembly               solvers.py:122-166
  * its LAPACK band LU + conditioning guard        solvers.py:168-186, 196-212
  * the forward operator (dt L + alpha) x          solvers.py:110-117, 214-237
  * the fixed pairwise pole reduction ``tree_sum`` steppers.py:157-172
  * ``realify_stacked``                            steppers.py:175-185
  * ``rexi_step``                                  steppers.py:214-235

(all paths relative to /root/reference/pkg/src/swerexi/).  Arrays are the
reference's dense ``(3, T+1, T+1)`` complex128 stacks [phi', vort, div].
"""

from __future__ import annotations

import dataclasses

import numpy as np
from scipy.linalg import lapack

KL = KU = 4            # solvers.py:23-24
COND_LIMIT = 1e13      # solvers.py:25


class OracleSolverError(RuntimeError):
    """Mirror of swerexi.errors.SolverError (errors.py:24-25)."""


@dataclasses.dataclass(frozen=True)
class Model:
    trunc: int
    phibar: float
    radius: float = 6.37122e6      # sphere.py:26
    omega: float = 7.292e-5        # sphere.py:27

    @property
    def kappa(self) -> np.ndarray:
        l = np.arange(self.trunc + 1, dtype=float)
        return l * (l + 1.0) / self.radius**2   # solvers.py:77


# ----------------------------------------------------------------------
# gravity group: diagonal per (l, m)

def lg_solutions(model: Model, dt: float, alphas, stack: np.ndarray) -> np.ndarray:
    """(N, 3, n, n) solutions of (dt L_g + alpha_n) x = b (solvers.py:86-108)."""
    alphas = np.asarray(alphas, dtype=np.complex128)
    a = alphas[:, None, None]
    kap = model.kappa[None, :, None]
    g = dt * dt * model.phibar * kap
    det = a * a + g
    bad = np.abs(det) <= 1e-13 * (np.abs(a) ** 2 + g)
    if bad.any():
        k, l, _ = np.argwhere(bad)[0]
        raise OracleSolverError(f"singular gravity block l={l} alpha={alphas[k]}")
    if np.any(alphas == 0):
        raise OracleSolverError("alpha = 0")
    bp, bz, bd = stack
    phi = (a * bp[None] + dt * model.phibar * bd[None]) / det
    div = (-dt * kap * bp[None] + a * bd[None]) / det
    vort = np.broadcast_to(bz[None] / a, phi.shape)
    return np.stack([phi, vort, div], axis=1)


def lg_apply(model: Model, dt: float, alpha: complex, stack: np.ndarray) -> np.ndarray:
    """(dt L_g + alpha) x  (solvers.py:110-117)."""
    bp, bz, bd = stack
    kap = model.kappa[:, None]
    return np.stack([alpha * bp - dt * model.phibar * bd, alpha * bz,
                     dt * kap * bp + alpha * bd])


# ----------------------------------------------------------------------
# Coriolis group: banded per zonal wavenumber m, unknowns interleaved
# p = 3k + {phi', vort, div}, l = m + k (solvers.py:122-166)

def _eps(l: np.ndarray, m: int) -> np.ndarray:
    l = np.asarray(l, dtype=float)
    num = l * l - m * m
    out = np.zeros_like(l)
    ok = num > 0
    out[ok] = np.sqrt(num[ok] / (4.0 * l[ok] * l[ok] - 1.0))
    return out


def l_band(model: Model, dt: float, m: int, coriolis: bool = True) -> np.ndarray:
    """dt*L for column m in LAPACK band storage (2KL+KU+1, 3(T+1-m))."""
    T = model.trunc
    nl = T + 1 - m
    size = 3 * nl
    ab = np.zeros((2 * KL + KU + 1, size), dtype=np.complex128)
    row0 = KL + KU                       # band row of the main diagonal
    ls = np.arange(m, T + 1)
    k = ls - m
    p = 3 * k
    kap = model.kappa[ls]
    w = dt * 2.0 * model.omega
    # entry (i, j) lives at ab[row0 + i - j, j]
    ab[row0 - 2, p + 2] += -dt * model.phibar           # phi'_l <- div_l
    ab[row0 + 2, p] += dt * kap                         # div_l  <- phi'_l
    if not (coriolis and model.omega > 0.0):
        return ab
    eps = _eps(np.arange(T + 2), m)
    pos = ls >= 1
    rot = np.zeros(nl, dtype=np.complex128)
    rot[pos] = w * 1j * m / (ls[pos] * (ls[pos] + 1.0))
    ab[row0, p + 1] += rot                              # vort diagonal
    ab[row0, p + 2] += rot                              # div diagonal
    lo = k >= 1                                          # couplings to l-1
    fac = np.where(ls - 1 >= 1, (ls + 1.0) / np.maximum(ls, 1), 1.0)
    c_lo = w * eps[ls] * fac
    ab[row0 + 2, (p - 1)[lo]] += -c_lo[lo]             # vort_l <- div_{l-1}
    ab[row0 + 4, (p - 2)[lo]] += c_lo[lo]              # div_l  <- vort_{l-1}
    hi = k + 1 < nl                                      # couplings to l+1
    c_hi = w * eps[np.minimum(ls + 1, T + 1)] * (ls / (ls + 1.0))
    ab[row0 - 4, (p + 5)[hi]] += -c_hi[hi]             # vort_l <- div_{l+1}
    ab[row0 - 2, (p + 4)[hi]] += c_hi[hi]              # div_l  <- vort_{l+1}
    return ab


class LFactors:
    """Per-(m, alpha) LU cache with the reference's guard (solvers.py:168-186)."""

    def __init__(self, model: Model, dt: float):
        self.model = model
        self.dt = dt
        self.bands = [l_band(model, dt, m) for m in range(model.trunc + 1)]
        self.norms = [float(np.max(np.sum(np.abs(b[KL:, :]), axis=0))) for b in self.bands]
        self.cache: dict = {}

    def factor(self, m: int, alpha: complex):
        key = (m, complex(alpha))
        hit = self.cache.get(key)
        if hit is not None:
            return hit
        ab = self.bands[m].copy()
        ab[KL + KU, :] += alpha
        lu, piv, info = lapack.zgbtrf(ab, KL, KU)
        if info != 0:
            raise OracleSolverError(f"band LU failed m={m} alpha={alpha} info={info}")
        dmin = float(np.min(np.abs(lu[KL + KU, :])))
        if dmin == 0.0 or (self.norms[m] + abs(alpha)) / dmin > COND_LIMIT:
            raise OracleSolverError(f"numerically singular band m={m} alpha={alpha}")
        self.cache[key] = (lu, piv)
        return lu, piv

    def solve(self, alpha: complex, stack: np.ndarray, keep: bool = True) -> np.ndarray:
        """(dt L + alpha)^-1 b for one shift (solvers.py:196-212)."""
        T = self.model.trunc
        out = np.zeros_like(stack)
        for m in range(T + 1):
            col = stack[:, m:, m]                      # (3, nl)
            rhs = np.ascontiguousarray(col.T).reshape(-1)   # interleaved 3k+f
            lu, piv = self.factor(m, alpha)
            x, info = lapack.zgbtrs(lu, KL, KU, rhs, piv)
            if info != 0:
                raise OracleSolverError(f"band solve failed m={m}")
            out[:, m:, m] = x.reshape(-1, 3).T
        if not keep:
            self.cache.clear()
        return out

    def apply(self, alpha: complex, stack: np.ndarray) -> np.ndarray:
        """(dt L + alpha) x via the band (solvers.py:214-237).

        The reference slices ``ab[row, :n+off]`` even when n+off < 0 (the
        m = T column, n = 3 < KL), which raises; skip those empty diagonals.
        """
        T = self.model.trunc
        out = np.zeros_like(stack)
        for m in range(T + 1):
            x = np.ascontiguousarray(stack[:, m:, m].T).reshape(-1)
            ab = self.bands[m]
            n = x.size
            y = alpha * x
            for off in range(-KL, KU + 1):
                row = KL + KU - off
                if abs(off) >= n:
                    continue
                if off >= 0:
                    y[: n - off] += ab[row, off:n] * x[off:n]
                else:
                    y[-off:] += ab[row, : n + off] * x[: n + off]
            out[:, m:, m] = y.reshape(-1, 3).T
        return out


# ----------------------------------------------------------------------
# pole reduction

def tree_sum(terms: np.ndarray) -> np.ndarray:
    """Pairwise (0,1),(2,3),... reduction over axis 0, odd tail carried
    (steppers.py:157-172)."""
    arr = terms
    while arr.shape[0] > 1:
        n = arr.shape[0]
        pairs = arr[0 : n - 1 : 2] + arr[1:n:2]
        arr = np.concatenate([pairs, arr[n - 1 : n]]) if n % 2 else pairs
    return arr[0]


def realify(stack: np.ndarray) -> tuple[np.ndarray, float]:
    """Drop the m=0 imaginary residue (steppers.py:175-185)."""
    residue = float(np.max(np.abs(stack[..., :, 0].imag))) if stack.size else 0.0
    out = stack.copy()
    out[..., :, 0] = out[..., :, 0].real
    return out, residue


def rexi_sum(group: str, model: Model, dt: float, alphas, betas, stack: np.ndarray,
             factors: LFactors | None = None, chunk: int = 16,
             do_realify: bool = True) -> np.ndarray:
    """realify(tree_sum(beta_n * solve(alpha_n, b)))  (steppers.py:214-235).

    For the l group the poles are solved ``chunk`` at a time and the chunk
    sums are reduced by the same tree; for power-of-two N and chunk this is
    bitwise equal to the reference's one-shot tree.
    """
    alphas = np.asarray(alphas, dtype=np.complex128)
    betas = np.asarray(betas, dtype=np.complex128)
    if group == "lg":
        # power-of-two chunks reduced by the same tree == the one-shot tree
        ch = 256 if alphas.size > 256 and (alphas.size & (alphas.size - 1)) == 0 else alphas.size
        parts = [tree_sum(betas[s:s + ch, None, None, None]
                          * lg_solutions(model, dt, alphas[s:s + ch], stack))
                 for s in range(0, alphas.size, ch)]
        total = tree_sum(np.stack(parts))
    elif group == "l":
        if factors is None:
            factors = LFactors(model, dt)
        parts = []
        for s in range(0, alphas.size, chunk):
            sols = np.stack([factors.solve(a, stack, keep=False)
                             for a in alphas[s:s + chunk]])
            parts.append(tree_sum(betas[s:s + chunk, None, None, None] * sols))
        total = tree_sum(np.stack(parts))
    else:
        raise ValueError(group)
    if do_realify:
        total, _ = realify(total)
    return total


def rexi_partial(group: str, model: Model, dt: float, alphas, betas, stack,
                 lo: int, hi: int, factors: LFactors | None = None) -> np.ndarray:
    """Un-realified tree sum over the contiguous pole block [lo, hi)
    (the per-worker share of parallel.py:137-156)."""
    return rexi_sum(group, model, dt, np.asarray(alphas)[lo:hi],
                    np.asarray(betas)[lo:hi], stack, factors, do_realify=False)


# ----------------------------------------------------------------------
# equivalent two-chain form of the l system (SURVEY §8a row a5'), used by
# the tests to pin the kernel's formulation against the band oracle

def chain_coefficients(model: Model, dt: float, m: int):
    """Real couplings (L_l, U_l), rotation r_l and kappa_l for column m."""
    T = model.trunc
    ls = np.arange(m, T + 1)
    w = dt * 2.0 * model.omega
    eps = _eps(np.arange(T + 2), m)
    r = np.zeros(ls.size, dtype=np.complex128)
    r[ls >= 1] = w * 1j * m / (ls[ls >= 1] * (ls[ls >= 1] + 1.0))
    fac = np.where(ls >= 2, (ls + 1.0) / np.maximum(ls, 1), 1.0)
    lower = w * eps[ls] * fac
    lower[0] = 0.0
    upper = w * eps[np.minimum(ls + 1, T + 1)] * ls / (ls + 1.0)
    upper[-1] = 0.0
    return ls, lower, upper, r, model.kappa[ls]


def chain_solve(model: Model, dt: float, alpha: complex, stack: np.ndarray) -> np.ndarray:
    """Solve the l system as two scalar tridiagonal chains per m (Thomas,
    no pivoting) after eliminating phi'."""
    T = model.trunc
    out = np.zeros_like(stack)
    pb = model.phibar
    for m in range(T + 1):
        ls, lower, upper, r, kap = chain_coefficients(model, dt, m)
        nl = ls.size
        bphi, bvort, bdiv = stack[0, m:, m], stack[1, m:, m], stack[2, m:, m]
        for c in (0, 1):
            k = np.arange(nl)
            is_vort = ((k + c) % 2) == 0
            diag = alpha + r + np.where(is_vort, 0.0, dt * dt * pb * kap / alpha)
            sgn = np.where(is_vort, -1.0, 1.0)
            sub = sgn * lower
            sup = sgn * upper
            rhs = np.where(is_vort, bvort, bdiv - (dt * kap / alpha) * bphi)
            cp = np.zeros(nl, dtype=np.complex128)
            yp = np.zeros(nl, dtype=np.complex128)
            for i in range(nl):
                den = diag[i] - (sub[i] * cp[i - 1] if i else 0.0)
                cp[i] = sup[i] / den
                yp[i] = (rhs[i] - (sub[i] * yp[i - 1] if i else 0.0)) / den
            x = np.zeros(nl, dtype=np.complex128)
            x[-1] = yp[-1]
            for i in range(nl - 2, -1, -1):
                x[i] = yp[i] - cp[i] * x[i + 1]
            lz = ls[is_vort]
            ld = ls[~is_vort]
            out[1, lz, m] = x[is_vort]
            out[2, ld, m] = x[~is_vort]
            out[0, ld, m] = (bphi[~is_vort] + dt * pb * x[~is_vort]) / alpha
    return out
