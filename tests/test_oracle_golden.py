"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import rel_l2, rel_linf, rel_to_scale
from oracle import layout, rexi as orx, sht as osh, stepping as ost

G = 9.80616


def model(trunc, omega=7.292e-5):
    return orx.Model(trunc, 1e4 * G, omega=omega)


@pytest.mark.parametrize("p0,p1,n", [(10, 30, 16), (10, 30, 128), (10, 30, 256), (15, 60, 256),
                                     (10, 30, 1024), (10, 60, 1024)])
def test_coefficients_bitwise(golden_small, p0, p1, n):
    for k in (0, 1, 2):
        a, b = ost.contour_coeffs(k, float(p0), float(p1), n)
        tag = f"coef_p{p0}_{p1}_n{n}_psi{k}"
        assert np.array_equal(a, golden_small[tag + "_alpha"])
        assert np.max(np.abs(b - golden_small[tag + "_beta"])) <= 1e-15 * np.max(np.abs(b))


@pytest.mark.parametrize("n", [32, 96, 386])
def test_gauss_nodes_bitwise(golden_small, n):
    x, w = osh.gauss_nodes(n)
    assert np.array_equal(x, golden_small[f"gauss{n}_x"])
    assert np.array_equal(w, golden_small[f"gauss{n}_w"])


def test_legendre_tables(golden_small):
    g = osh.Grid(21)
    assert np.max(np.abs(g.P - golden_small["T21_P"])) < 1e-14
    assert np.max(np.abs(g.H - golden_small["T21_H"])) < 1e-13


def test_transforms_t21(golden_small):
    g = osh.Grid(21)
    st = layout.unpack(golden_small["T21_sht_in"], 21)
    assert rel_linf(g.synthesis(st[0]).ravel(), golden_small["T21_synth_phi"].ravel()) < 1e-13
    u, v = g.uv_from_vortdiv(st[1], st[2])
    assert rel_linf(u.ravel(), golden_small["T21_u"].ravel()) < 1e-13
    assert rel_linf(v.ravel(), golden_small["T21_v"].ravel()) < 1e-13
    grid = golden_small["T21_grid_in"]
    an = layout.pack(g.analysis(grid)[None])[0]
    assert rel_linf(an, golden_small["T21_analysis"]) < 1e-13
    z, d = g.vortdiv_from_uv(grid, grid[::-1].copy())
    assert rel_linf(layout.pack(z[None])[0], golden_small["T21_vd_z"]) < 1e-13
    assert rel_linf(layout.pack(d[None])[0], golden_small["T21_vd_d"]) < 1e-13


def test_tendencies_t21(golden_small):
    g = osh.Grid(21)
    st = layout.unpack(golden_small["T21_sht_in"], 21)
    assert rel_linf(layout.pack(g.tendency_lc(st)), golden_small["T21_tend_lc"]) < 1e-13
    assert rel_linf(layout.pack(g.tendency_n(st)), golden_small["T21_tend_n"]) < 1e-13
    assert rel_linf(layout.pack(g.tendency_lc_n(st)), golden_small["T21_tend_lc_n"]) < 1e-13


def test_tendency_t63(golden_small):
    g = osh.Grid(63)
    st = layout.unpack(golden_small["T63_sht_in"], 63)
    assert rel_linf(layout.pack(g.tendency_lc_n(st)), golden_small["T63_tend_lc_n"]) < 1e-12
    assert rel_linf(g.synthesis(st[0]).ravel(), golden_small["T63_synth_phi"].ravel()) < 1e-13


def test_seeded_inputs_match(golden_small, golden_medium):
    assert np.array_equal(layout.pack(ost.seeded_linear_state(63, 0)), golden_small["cfg0_in"])
    assert np.array_equal(layout.pack(ost.seeded_linear_state(128, 0)), golden_medium["cfg1_in"])
    ic = layout.pack(ost.seeded_balanced_state(osh.Grid(42)))
    assert rel_linf(ic, golden_medium["T42etd_ic"]) < 1e-13


def test_cfg0_lg_rexi(golden_small):
    a, b = ost.contour_coeffs(0, 10.0, 30.0, 128)
    st = layout.unpack(golden_small["cfg0_in"], 63)
    out = orx.rexi_sum("lg", model(63), 3600.0, a, b, st)
    assert np.array_equal(layout.pack(out), golden_small["cfg0_out"])


def test_l_rexi_t21_and_single(golden_small):
    a, b = ost.contour_coeffs(0, 10.0, 30.0, 16)
    st = layout.unpack(golden_small["T21_l16_in"], 21)
    m = model(21)
    out = orx.rexi_sum("l", m, 480.0, a, b, st)
    assert rel_linf(layout.pack(out), golden_small["T21_l16_out"]) < 1e-14
    assert np.array_equal(layout.pack(orx.rexi_sum("lg", m, 480.0, a, b, st)),
                          golden_small["T21_lg16_out"])
    fac = orx.LFactors(m, 480.0)
    assert rel_linf(layout.pack(fac.solve(1.3 - 0.8j, st)), golden_small["T21_l_single_out"]) < 1e-14
    assert np.array_equal(layout.pack(orx.lg_apply(m, 480.0, 0.7 + 0.2j, st)),
                          golden_small["T21_lg_apply_out"])


def test_chain_form_equals_band(golden_small):
    """The two-chain Thomas form the CUDA kernel uses reproduces the
    reference band solve (SURVEY §8a row a5')."""
    st = layout.unpack(golden_small["T21_l16_in"], 21)
    m = model(21)
    x = orx.chain_solve(m, 480.0, 1.3 - 0.8j, st)
    assert rel_linf(layout.pack(x), golden_small["T21_l_single_out"]) < 1e-13


def test_l_rexi_t42(golden_small):
    a, b = ost.contour_coeffs(0, 10.0, 30.0, 128)
    st = layout.unpack(golden_small["T42_l128_in"], 42)
    out = orx.rexi_sum("l", model(42), 3600.0, a, b, st)
    assert rel_linf(layout.pack(out), golden_small["T42_l128_out"]) < 1e-13


def test_etdrk_t42_trajectory(golden_medium):
    g = osh.Grid(42)
    m = model(42)
    sets = {k: ost.contour_coeffs(k, 10.0, 30.0, 128) for k in (0, 1, 2)}
    st = layout.unpack(golden_medium["T42etd_ic"], 42)
    st = ost.etdrk2_step(m, g, 1800.0, sets, st)
    assert rel_linf(layout.pack(st), golden_medium["T42etd_step1"]) < 1e-12
    for _ in range(7):
        st = ost.etdrk2_step(m, g, 1800.0, sets, st)
    assert rel_l2(layout.pack(st), golden_medium["T42etd_step8"]) < 1e-11


@pytest.mark.slow
def test_cfg1_l_rexi(golden_medium):
    a, b = ost.contour_coeffs(0, 10.0, 30.0, 256)
    st = layout.unpack(golden_medium["cfg1_in"], 128)
    out = orx.rexi_sum("l", model(128), 7200.0, a, b, st)
    assert rel_linf(layout.pack(out), golden_medium["cfg1_out"]) < 1e-12


# ---------------------------------------------------------------- T1279 / T383
# fixtures from tests/golden/make_golden_large.py (the reference run on the
# pieces of the large problems it can hold)

def _load(name):
    import os

    from conftest import GOLDEN
    return np.load(os.path.join(GOLDEN, name))


@pytest.mark.parametrize("m", [640, 1279])
def test_oracle_cfg4_columns_all_poles(m):
    """The oracle's band LU + tree over all 1024 cfg4 poles on column m
    equals the reference's (solvers.py:168-212, steppers.py:157-172)."""
    gold = _load("l1279.npz")
    trunc = 1279
    fac = orx.LFactors(model(trunc), 14400.0)
    st = ost.seeded_linear_state(trunc, 0)
    a, b = gold["alphas"], gold["betas"]
    col = np.ascontiguousarray(st[:, m:, m].T).reshape(-1)
    terms = []
    for k in range(a.size):
        lu, piv = fac.factor(m, a[k])
        x, info = orx.lapack.zgbtrs(lu, orx.KL, orx.KU, col, piv)
        assert info == 0
        fac.cache.clear()
        terms.append(b[k] * x.reshape(-1, 3).T)
    for i, k in enumerate(gold["poles"]):  # single solves: no cancellation
        assert rel_linf(terms[k], gold[f"poles_m{m}"][i]) <= 1e-12
    got = orx.tree_sum(np.stack(terms))
    assert rel_to_scale(got, gold[f"sum_m{m}"], gold[f"abs_m{m}"]) <= 1e-13


def test_oracle_t1279_legendre_chunks():
    """Oracle tables on the T1279 latitude chunks reproduce the reference's
    chunked synthesis rows and analysis columns (sphere.py:72-112, 297-347)."""
    gold = _load("sht1279.npz")
    trunc, nlon = 1279, 3840
    x = gold["x"]
    xo, wo = osh.gauss_nodes(1920)
    assert np.array_equal(xo, x) and np.array_equal(wo, gold["w"])
    spec = ost.seeded_linear_state(trunc, 0)[0]
    for j0, j1 in gold["chunks"]:
        P, _ = osh.legendre_tables(trunc, x[j0:j1])
        P = P[:, : trunc + 1, :]
        g = np.einsum("jlm,lm->jm", P, spec)
        half = np.zeros((j1 - j0, nlon // 2 + 1), dtype=np.complex128)
        half[:, : trunc + 1] = g
        rows = np.fft.irfft(half, n=nlon, axis=1) * nlon
        assert rel_linf(rows.ravel(), gold[f"synth_{j0}"].ravel()) <= 1e-12
        four = np.fft.fft(gold[f"grid_{j0}"], axis=1) * (2 * np.pi / nlon)
        fw = four[:, : trunc + 1] * gold["w"][j0:j1, None]
        for m in gold["cols"]:
            c = np.einsum("jl,j->l", P[:, m:, m], fw[:, m])
            assert rel_linf(c, gold[f"ana_{j0}_m{m}"]) <= 1e-12
