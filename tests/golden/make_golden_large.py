"""Golden fixtures for the large-truncation range (T383 and T1279), produced by
running the REFERENCE itself on the pieces of the problem it can hold in memory.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_large.py [--l1279] [--sht1279] [--etd383]

* ``--l1279`` (cfg4, l_rexi T1279, N=1024, dt=14400, seeded linear state):
  the l system is independent per zonal wavenumber m (solvers.py:196-212), so
  the reference's own band LU (``ShiftedLinearSolver._factor`` / zgbtrs) is run
  for ALL 1024 poles on the columns m in {0, 1, 2, 640, 1279} only.  The
  solver's ``plan_for`` call is shimmed to the single array it reads (``ll1``,
  solvers.py:76-77); the factor cache is cleared per pole.
  Stored: the beta-weighted ``tree_sum`` (steppers.py:157-172) over all 1024
  poles per column (unrealified), the entrywise sum of |beta_n x_n| (the sums
  cancel by up to 1e10 on this contour, so their rounding floor is relative to
  that scale, not to the sum), and the individual beta-weighted solves of
  the poles around the contour's imaginary-axis crossings (n = 100..111 and
  912..923, the least diagonally dominant chains).
* ``--sht1279``: T1279 transforms on latitude chunks.  The
  reference's own ``gauss_legendre_nodes(1920)`` and ``_legendre_tables(1279,
  x[j0:j1])`` build the tables of three chunks (polar, mid-latitude,
  equator-straddling); the reference's ``SpherePlan.synth_cols`` /
  ``analyze_cols`` and ``_real_fourier_synth`` run unchanged on a plan object
  restricted to the chunk.  Synthesis is row-local, so the chunk rows equal
  the full transform's rows; analysis is linear in the grid, so a grid that
  is zero outside the chunk gives exactly the chunk's quadrature sum.
* ``--etd383``: two ETD2RK steps of ``lg_rexi_lc_n_etdrk`` at T383 (the
  cuFFT / column-walk / table path above T341), N=256, dt=1200 s, seeded
  balanced state (as cfg2).
"""

from __future__ import annotations

import argparse
import os
import sys
import time
from types import SimpleNamespace

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from make_golden import pack, seeded_balanced_state, seeded_linear_state  # noqa: E402
from swerexi import rexi as R  # noqa: E402
from swerexi import solvers as S  # noqa: E402
from swerexi import sphere as SP  # noqa: E402
from swerexi import steppers as ST  # noqa: E402
from swerexi import swe as W  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
L1279_COLS = (0, 1, 2, 640, 1279)
L1279_POLES = tuple(range(100, 112)) + tuple(range(912, 924))
SHT_CHUNKS = ((0, 8), (480, 488), (956, 964))
SHT_COLS = (0, 1, 640, 1279)


def l1279(path):
    trunc = 1279
    cfg = SP.SphereConfig.for_truncation(trunc)
    par = W.ModelParams(1e4 * cfg.gravity_g, cfg)
    ll1 = np.arange(trunc + 1) * (np.arange(trunc + 1) + 1.0)
    S.plan_for = lambda c: SimpleNamespace(ll1=ll1)  # only .ll1 is read (solvers.py:76-77)
    sol = S.ShiftedLinearSolver(W.L, 14400.0, par)
    coeffs = R.RexiSetup(num_poles=1024).coefficients("psi0", 14400.0)
    st = seeded_linear_state(trunc, 0)
    out = {"alphas": coeffs.alphas, "betas": coeffs.betas}
    t0 = time.time()
    for m in L1279_COLS:
        nl = trunc + 1 - m
        rhs = np.empty(3 * nl, dtype=np.complex128)
        rhs[0::3], rhs[1::3], rhs[2::3] = st[0, m:, m], st[1, m:, m], st[2, m:, m]
        terms = np.empty((coeffs.num_terms, 3, nl), dtype=np.complex128)
        for k, (a, b) in enumerate(zip(coeffs.alphas, coeffs.betas)):
            lu, piv = sol._factor(m, a)
            x, info = S.lapack.zgbtrs(lu, S._KL, S._KU, rhs, piv)
            assert info == 0
            sol._factors.clear()
            terms[k, 0], terms[k, 1], terms[k, 2] = x[0::3], x[1::3], x[2::3]
            terms[k] *= b  # steppers.py:232
        out[f"sum_m{m}"] = ST.tree_sum(terms)
        out[f"abs_m{m}"] = np.abs(terms).sum(axis=0)  # summation scale (cancellation)
        out[f"poles_m{m}"] = terms[list(L1279_POLES)]
        print(f"m={m}: {time.time() - t0:.1f}s", flush=True)
    out["poles"] = np.array(L1279_POLES)
    out["cols"] = np.array(L1279_COLS)
    np.savez_compressed(path, **out)


def _chunk_plan(trunc, nlon, x, w, j0, j1):
    """A SpherePlan restricted to latitudes [j0, j1): the reference's own
    table builder on the chunk, the attribute layout of SpherePlan.__init__
    (sphere.py:174-197) so its synth_cols/analyze_cols methods run as-is."""
    p_ext, h = SP._legendre_tables(trunc, x[j0:j1])
    p = np.ascontiguousarray(p_ext[:, : trunc + 1, :])
    plan = SimpleNamespace()
    plan._ana = {"p": np.ascontiguousarray(p.transpose(2, 1, 0))}
    plan._syn = {"p": np.ascontiguousarray(p.transpose(2, 0, 1))}
    plan.weights = w[j0:j1]
    plan.dlon = 2.0 * np.pi / nlon
    return plan


def sht1279(path):
    trunc = 1279
    cfg = SP.SphereConfig.for_truncation(trunc)
    x, w = SP.gauss_legendre_nodes(cfg.nlat)
    spec = seeded_linear_state(trunc, 0)[0]  # the cfg4 Phi' field (real origin)
    rng = np.random.default_rng(11)
    out = {"x": x, "w": w, "chunks": np.array(SHT_CHUNKS), "cols": np.array(SHT_COLS)}
    nm = trunc + 1
    for j0, j1 in SHT_CHUNKS:
        t0 = time.time()
        plan = _chunk_plan(trunc, cfg.nlon, x, w, j0, j1)
        g = SP.SpherePlan.synth_cols(plan, spec, "p")  # sphere.py:332
        out[f"synth_{j0}"] = SP._real_fourier_synth(g, cfg.nlon)  # sphere.py:342-347
        grid = rng.standard_normal((j1 - j0, cfg.nlon))
        fourier = np.fft.fft(grid, axis=1) * plan.dlon  # sphere.py:306
        coeffs = SP.SpherePlan.analyze_cols(plan, fourier[:, :nm], "p", plan.weights)
        out[f"grid_{j0}"] = grid
        for m in SHT_COLS:
            out[f"ana_{j0}_m{m}"] = coeffs[m:, m].copy()
        print(f"chunk {j0}: {time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(path, **out)


def etd383(path, steps=2):
    trunc, dt = 383, 1200.0
    cfg = SP.SphereConfig.for_truncation(trunc)
    par = W.ModelParams(1e4 * cfg.gravity_g, cfg)
    s = seeded_balanced_state(cfg)
    out = {"ic": pack(s.stack()), "dt": np.array(dt)}
    stepper = ST.build_stepper("lg_rexi_lc_n_etdrk", par, R.RexiSetup(num_poles=256))
    t0 = time.time()
    for k in range(1, steps + 1):
        s = stepper.step(s, dt)
        out[f"step{k}"] = pack(s.stack())
        print(f"T383 step {k}: {time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(path, **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--l1279", action="store_true")
    ap.add_argument("--sht1279", action="store_true")
    ap.add_argument("--etd383", action="store_true")
    a = ap.parse_args()
    if a.l1279:
        l1279(os.path.join(HERE, "l1279.npz"))
    if a.sht1279:
        sht1279(os.path.join(HERE, "sht1279.npz"))
    if a.etd383:
        etd383(os.path.join(HERE, "etd383.npz"))


if __name__ == "__main__":
    main()
