"""Generate golden fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--big]

Every array written here comes out of ``swerexi`` (the reference package,
imported read-only from /root/reference/pkg/src); the seeded inputs follow
SURVEY §8(d).  Spectral states are stored packed m-major (the reference's
``mode_index_map`` order, solvers.py:288-290) as complex128.  The GPU box
never runs this script; it only reads the .npz files it wrote.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from swerexi import rexi as R  # noqa: E402
from swerexi import solvers as S  # noqa: E402
from swerexi import sphere as SP  # noqa: E402
from swerexi import steppers as ST  # noqa: E402
from swerexi import swe as W  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def pack(stack):
    t = stack.shape[-1] - 1
    idx = S.mode_index_map(t)
    l = np.array([a for a, _ in idx])
    m = np.array([b for _, b in idx])
    return np.ascontiguousarray(stack[..., l, m])


def seeded_linear_state(trunc, seed=0):
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


def seeded_balanced_state(cfg, peak=1e-5, seed=0):
    rng = np.random.default_rng(seed)
    n = cfg.trunc + 1
    l = np.arange(n)[:, None]
    m = np.arange(n)[None, :]
    c = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / (l + 1.0) ** 1.5
    c[m > l] = 0.0
    c[:, 0] = c[:, 0].real
    c[0, 0] = 0.0
    zmax = np.max(np.abs(SP.synthesis(SP.SpectralField(c), cfg).values))
    c = c * (peak / zmax)
    st = W.PrognosticState.zeros(cfg)
    st.vort.coeffs[:] = c
    params = W.ModelParams(1e4 * cfg.gravity_g, cfg)
    lc = W.tendency_lc(st, params)
    kap = SP.plan_for(cfg).ll1 / cfg.radius_a**2
    phi = np.zeros((n, n), dtype=np.complex128)
    phi[1:] = -lc.div.coeffs[1:] / kap[1:, None]
    st.phi_pert.coeffs[:] = phi
    return st


def state_of(stack, cfg):
    return W.PrognosticState.from_stack(stack, cfg)


def coeff_fixtures(out):
    for (p0, p1, n) in [(10.0, 30.0, 16), (10.0, 30.0, 128), (10.0, 30.0, 256),
                        (15.0, 60.0, 256), (10.0, 30.0, 1024), (10.0, 60.0, 1024)]:
        con = R.shifted_contour_from_points(p0, p1, n)
        for k in (0, 1, 2):
            c = R.coeffs_for_contour(f"psi{k}", con)
            tag = f"coef_p{int(p0)}_{int(p1)}_n{n}_psi{k}"
            out[tag + "_alpha"] = c.alphas
            out[tag + "_beta"] = c.betas


def sht_fixtures(out):
    for n in (32, 96, 386):
        x, w = SP.gauss_legendre_nodes(n)
        out[f"gauss{n}_x"] = x
        out[f"gauss{n}_w"] = w
    cfg = SP.SphereConfig.for_truncation(21)
    plan = SP.plan_for(cfg)
    out["T21_P"] = plan.p
    out["T21_H"] = plan.h
    st = seeded_linear_state(21, seed=5)
    params = W.ModelParams(1e4 * cfg.gravity_g, cfg)
    s = state_of(st, cfg)
    out["T21_sht_in"] = pack(st)
    out["T21_synth_phi"] = SP.synthesis(s.phi_pert, cfg).values
    u, v = SP.uv_from_vortdiv(s.vort, s.div, cfg)
    out["T21_u"] = u.values
    out["T21_v"] = v.values
    grid = np.random.default_rng(7).standard_normal((cfg.nlat, cfg.nlon))
    out["T21_grid_in"] = grid
    out["T21_analysis"] = pack(SP.analysis(SP.GridField(grid, cfg), cfg).coeffs[None])[0]
    z, d = SP.vortdiv_from_uv(SP.GridField(grid, cfg), SP.GridField(grid[::-1].copy(), cfg), cfg)
    out["T21_vd_z"] = pack(z.coeffs[None])[0]
    out["T21_vd_d"] = pack(d.coeffs[None])[0]
    out["T21_tend_lc"] = pack(W.tendency_lc(s, params).stack())
    out["T21_tend_n"] = pack(W.tendency_n(s, params).stack())
    out["T21_tend_lc_n"] = pack(W.tendency_group(W.LC_N, s, params).stack())
    # larger transform case at the cfg0 grid
    cfg63 = SP.SphereConfig.for_truncation(63)
    st63 = seeded_linear_state(63, seed=6)
    s63 = state_of(st63, cfg63)
    out["T63_sht_in"] = pack(st63)
    out["T63_tend_lc_n"] = pack(
        W.tendency_group(W.LC_N, s63, W.ModelParams(1e4 * cfg63.gravity_g, cfg63)).stack())
    out["T63_synth_phi"] = SP.synthesis(s63.phi_pert, cfg63).values


def linear_fixtures(out):
    # cfg0: lg_rexi T63, N=128, dt=3600
    cfg = SP.SphereConfig.for_truncation(63)
    par = W.ModelParams(1e4 * cfg.gravity_g, cfg)
    st = seeded_linear_state(63, seed=0)
    coeffs = R.RexiSetup(num_poles=128).coefficients("psi0", 3600.0)
    res = ST.rexi_step(W.LG, state_of(st, cfg), 3600.0, coeffs, par)
    out["cfg0_in"] = pack(st)
    out["cfg0_out"] = pack(res.stack())
    # small l cases
    cfg21 = SP.SphereConfig.for_truncation(21)
    par21 = W.ModelParams(1e4 * cfg21.gravity_g, cfg21)
    st21 = seeded_linear_state(21, seed=1)
    c16 = R.coeffs_for_contour("psi0", R.shifted_contour_from_points(10.0, 30.0, 16))
    out["T21_l16_in"] = pack(st21)
    out["T21_l16_out"] = pack(ST.rexi_step(W.L, state_of(st21, cfg21), 480.0, c16, par21).stack())
    out["T21_lg16_out"] = pack(ST.rexi_step(W.LG, state_of(st21, cfg21), 480.0, c16, par21).stack())
    sol = S.ShiftedLinearSolver(W.L, 480.0, par21)
    out["T21_l_single_out"] = pack(sol.solve_stacked(1.3 - 0.8j, st21))
    # NB: ShiftedLinearSolver.apply_stacked for group 'l' raises at m = T
    # (solvers.py:231-233 slices ab[row, :n+off] with n+off < 0); pin lg only.
    out["T21_lg_apply_out"] = pack(S.ShiftedLinearSolver(W.LG, 480.0, par21).apply_stacked(0.7 + 0.2j, st21))
    # l_rexi at T42, N=128, dt=3600
    cfg42 = SP.SphereConfig.for_truncation(42)
    par42 = W.ModelParams(1e4 * cfg42.gravity_g, cfg42)
    st42 = seeded_linear_state(42, seed=2)
    c128 = R.RexiSetup(num_poles=128).coefficients("psi0", 3600.0)
    out["T42_l128_in"] = pack(st42)
    out["T42_l128_out"] = pack(ST.rexi_step(W.L, state_of(st42, cfg42), 3600.0, c128, par42).stack())


def cfg1_fixture(out):
    # cfg1: l_rexi T128 (194x388), N=256, dt=7200, default contour
    cfg = SP.SphereConfig.for_truncation(128)
    par = W.ModelParams(1e4 * cfg.gravity_g, cfg)
    st = seeded_linear_state(128, seed=0)
    coeffs = R.RexiSetup(num_poles=256).coefficients("psi0", 7200.0)
    t0 = time.time()
    res = ST.rexi_step(W.L, state_of(st, cfg), 7200.0, coeffs, par)
    print(f"cfg1 reference step {time.time() - t0:.1f}s")
    out["cfg1_in"] = pack(st)
    out["cfg1_out"] = pack(res.stack())


def etdrk_fixtures(out, trunc, steps, tag, dt=1800.0, n_poles=256):
    cfg = SP.SphereConfig.for_truncation(trunc)
    par = W.ModelParams(1e4 * cfg.gravity_g, cfg)
    s = seeded_balanced_state(cfg)
    out[f"{tag}_ic"] = pack(s.stack())
    stepper = ST.build_stepper("lg_rexi_lc_n_etdrk", par, R.RexiSetup(num_poles=n_poles))
    t0 = time.time()
    for k in range(1, steps + 1):
        s = stepper.step(s, dt)
        if k == 1 or k == steps:
            out[f"{tag}_step{k}"] = pack(s.stack())
    print(f"{tag}: {steps} ETD2RK steps in {time.time() - t0:.1f}s")


def split_fixtures(path):
    """Strang-split (ERK2 + REXI / CN) and CN steppers at T21 (rows f2/f3)."""
    out = {}
    cfg = SP.SphereConfig.for_truncation(21)
    par = W.ModelParams(1e4 * cfg.gravity_g, cfg)
    s0 = seeded_balanced_state(cfg)
    out["T21split_ic"] = pack(s0.stack())
    for sid in ("lg_rexi_lc_n_erk_ver1", "lg_irk_lc_n_erk_ver0", "ln_erk"):
        st = ST.build_stepper(sid, par, R.RexiSetup(num_poles=64))
        s = s0
        for _ in range(2):
            s = st.step(s, 600.0)
        out[f"T21split_{sid}"] = pack(s.stack())
    np.savez_compressed(path, **out)


def io_fixtures(path):
    """f4: vorticity/divergence from grid winds, the Galewsky jet initial
    state, the L-inf error metric and the byte format of field dumps."""
    import io as _io

    from swerexi import benchmarks as B
    from swerexi import fieldio as FIO

    out = {}
    for trunc in (21, 42):
        cfg = SP.SphereConfig.for_truncation(trunc)
        src = seeded_linear_state(trunc, 7)
        u, v = SP.uv_from_vortdiv(SP.SpectralField(src[1]), SP.SpectralField(src[2]), cfg)
        z, d = SP.vortdiv_from_uv(u, v, cfg)
        out[f"T{trunc}_u"] = u.values
        out[f"T{trunc}_v"] = v.values
        out[f"T{trunc}_vort"] = pack(z.coeffs)
        out[f"T{trunc}_div"] = pack(d.coeffs)
    cfg = SP.SphereConfig.for_truncation(42)
    st = B.init_barotropic_instability(cfg, with_bump=True)
    out["T42_galewsky"] = pack(st.stack())
    st0 = B.init_barotropic_instability(cfg, with_bump=False)
    out["T42_galewsky_nobump"] = pack(st0.stack())
    out["T42_linf_h"] = np.array(B.linf_error(st, st0, "h"))
    out["T42_linf_vort"] = np.array(B.linf_error(st, st0, "vort"))
    # byte format of a two-block spectral dump and one grid block (T5 state)
    cfg5 = SP.SphereConfig.for_truncation(5)
    s5 = seeded_linear_state(5, 3)
    buf = _io.BytesIO()
    for f in range(3):
        FIO.write_spectral_block(buf, SP.SpectralField(s5[f]), cfg5)
    g = SP.synthesis(SP.SpectralField(s5[0]), cfg5)
    FIO.write_grid_block(buf, g, cfg5)
    out["T5_dump_bytes"] = np.frombuffer(buf.getvalue(), dtype=np.uint8)
    out["T5_state"] = pack(s5)
    out["T5_grid"] = g.values
    np.savez_compressed(path, **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also the T256 one-day trajectory")
    ap.add_argument("--split", action="store_true", help="only the Strang/CN stepper fixtures")
    ap.add_argument("--io", action="store_true", help="only the f4 (IC / error / dump) fixtures")
    args = ap.parse_args()
    if args.io:
        io_fixtures(os.path.join(HERE, "io.npz"))
        return
    if args.split:
        split_fixtures(os.path.join(HERE, "split.npz"))
        return
    out: dict = {}
    coeff_fixtures(out)
    sht_fixtures(out)
    linear_fixtures(out)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
    out = {}
    cfg1_fixture(out)
    etdrk_fixtures(out, 42, 8, "T42etd", n_poles=128)
    np.savez_compressed(os.path.join(HERE, "medium.npz"), **out)
    if args.big:
        out = {}
        etdrk_fixtures(out, 256, 48, "T256etd", n_poles=256)
        np.savez_compressed(os.path.join(HERE, "cfg2.npz"), **out)


if __name__ == "__main__":
    main()
