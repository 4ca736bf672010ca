"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden vectors and the CPU oracle.  Bars (BASELINE.json north star):
linear REXI steps relative L-inf <= 1e-10 per field, ETD2RK trajectories
relative L2 <= 1e-8 after one simulated day."""

import numpy as np
import pytest

from conftest import rel_l2, rel_linf

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import layout as olay  # noqa: E402
from oracle import rexi as orx  # noqa: E402
from oracle import sht as osh  # noqa: E402
from oracle import stepping as ost  # noqa: E402
from paper_1805_06557_b200 import _lib  # noqa: E402
from paper_1805_06557_b200.device import pack, ptr, stream_ptr, to_device, unpack  # noqa: E402
from paper_1805_06557_b200.errors import SolverError  # noqa: E402
from paper_1805_06557_b200.rexi import RexiSetup, coeffs_for_contour, shifted_contour_from_points  # noqa: E402
from paper_1805_06557_b200.solvers import ShiftedLinearSolver  # noqa: E402
from paper_1805_06557_b200.sphere import SphereConfig, plan_for  # noqa: E402
from paper_1805_06557_b200.steppers import (EtdrkStepper, build_stepper,  # noqa: E402
                                            integrate, rexi_step)
from paper_1805_06557_b200.swe import L, LC_N, LG, ModelParams, PrognosticState  # noqa: E402

G = 9.80616
LIN_BAR = 1e-10


def params(trunc, omega=7.292e-5):
    cfg = SphereConfig.for_truncation(trunc, omega=omega)
    return ModelParams(1e4 * G, cfg)


def coeffs(n, k=0, p0=10.0, p1=30.0):
    return coeffs_for_contour(f"psi{k}", shifted_contour_from_points(p0, p1, n))


def run_rexi(group, trunc, dt, n, packed_in, p0=10.0, p1=30.0):
    par = params(trunc)
    c = coeffs(n, 0, p0, p1)
    st = PrognosticState.from_stack(unpack(packed_in, trunc), par.cfg)
    out = rexi_step(group, st, dt, c, par)
    return pack(out.stack())


# ---------------------------------------------------------------- linear REXI

def test_cfg0_lg_rexi_golden(golden_small):
    out = run_rexi(LG, 63, 3600.0, 128, golden_small["cfg0_in"])
    assert rel_linf(out, golden_small["cfg0_out"]) <= LIN_BAR
    assert np.all(out[:, :64].imag == 0.0)  # realified m = 0 column


def test_t21_lg_and_l_golden(golden_small):
    for group, key in ((LG, "T21_lg16_out"), (L, "T21_l16_out")):
        out = run_rexi(group, 21, 480.0, 16, golden_small["T21_l16_in"])
        assert rel_linf(out, golden_small[key]) <= LIN_BAR, key


def test_t42_l_golden(golden_small):
    out = run_rexi(L, 42, 3600.0, 128, golden_small["T42_l128_in"])
    assert rel_linf(out, golden_small["T42_l128_out"]) <= LIN_BAR


def test_cfg1_l_rexi_golden(golden_medium):
    out = run_rexi(L, 128, 7200.0, 256, golden_medium["cfg1_in"])
    assert rel_linf(out, golden_medium["cfg1_out"]) <= LIN_BAR


def test_cfg1_accuracy_variant_vs_oracle():
    """p0=15, p1=60 contour (max|beta| 1.6e6, summation floor 1.5e-11)."""
    st = ost.seeded_linear_state(128, 0)
    a, b = ost.contour_coeffs(0, 15.0, 60.0, 256)
    ref = olay.pack(orx.rexi_sum("l", orx.Model(128, 1e4 * G), 7200.0, a, b, st, chunk=64))
    out = run_rexi(L, 128, 7200.0, 256, olay.pack(st), 15.0, 60.0)
    assert rel_linf(out, ref) <= LIN_BAR


def test_single_solve_and_apply(golden_small):
    par = params(21)
    st = unpack(golden_small["T21_l16_in"], 21)
    sl = ShiftedLinearSolver(L, 480.0, par)
    x = sl.solve_stacked(1.3 - 0.8j, st)
    assert rel_linf(pack(x), golden_small["T21_l_single_out"]) <= 1e-12
    # residual against the oracle's forward band operator
    fac = orx.LFactors(orx.Model(21, 1e4 * G), 480.0)
    res = fac.apply(1.3 - 0.8j, x) - st
    assert np.max(np.abs(res)) <= 1e-10 * np.max(np.abs(st))
    y = sl.apply_stacked(0.7 + 0.2j, st)
    assert rel_linf(pack(y), olay.pack(fac.apply(0.7 + 0.2j, st))) <= 1e-13
    slg = ShiftedLinearSolver(LG, 480.0, par)
    assert rel_linf(pack(slg.apply_stacked(0.7 + 0.2j, st)), golden_small["T21_lg_apply_out"]) <= 1e-14


def test_two_rhs_fusion_matches_separate():
    """n_rhs = 2 (ETD2RK psi0/psi1 fusion) equals two single sums."""
    par = params(42)
    for group in (LG, L):
        sl = ShiftedLinearSolver(group, 900.0, par)
        c0, c1 = coeffs(64, 0), coeffs(64, 1)
        u = ost.seeded_linear_state(42, 1)
        v = ost.seeded_linear_state(42, 2)
        rhs = to_device(np.stack([pack(u), pack(v)]))
        bet = to_device(np.stack([c0.betas, c1.betas]))
        out = sl.rexi_sum_dev(c0.alphas, bet, rhs).cpu().numpy()
        model = orx.Model(42, 1e4 * G)
        for r, (st, c) in enumerate(((u, c0), (v, c1))):
            ref = olay.pack(orx.rexi_sum(group.token, model, 900.0, c.alphas, c.betas, st))
            assert rel_linf(out[r], ref) <= LIN_BAR


@pytest.mark.parametrize("group", ["lg", "l"])
def test_pole_blocks_combine_bitwise(group):
    """Per-rank partials over aligned power-of-two pole blocks, combined by
    the fixed tree, equal the one-launch sum bitwise for K = 1, 2, 4, 8
    (test_parallel.py:67-78 analogue, emulated on one GPU)."""
    par = params(63)
    sl = ShiftedLinearSolver(L if group == "l" else LG, 3600.0, par)
    c = coeffs(256)
    rhs = to_device(pack(ost.seeded_linear_state(63, 3)))[None]
    bet = to_device(c.betas.reshape(1, -1))
    full = sl.rexi_sum_dev(c.alphas, bet, rhs).cpu().numpy()
    lib = _lib.load()
    for k in (2, 4, 8):
        parts = torch.stack([sl.rexi_sum_dev(c.alphas, bet, rhs, pole_range=(r * 256 // k, (r + 1) * 256 // k),
                                             realify=False) for r in range(k)]).contiguous()
        out = torch.empty_like(rhs)
        _lib.check(lib.swx_tree_combine(63, 1, k, ptr(parts), 1, ptr(out), stream_ptr()))
        assert np.array_equal(out.cpu().numpy(), full), k


def test_singular_shifts_raise():
    par = params(21)
    l = 7
    kappa = l * (l + 1) / par.cfg.radius_a**2
    alpha = 1j * 480.0 * np.sqrt(par.mean_geopotential * kappa)
    with pytest.raises(SolverError):
        ShiftedLinearSolver(LG, 480.0, par).warm(np.array([1.0 + 1j, alpha]))
    with pytest.raises(SolverError):
        ShiftedLinearSolver(LG, 480.0, par).warm(np.array([0.0 + 0j]))
    # band operator eigenvalue -> singular Coriolis system
    p10 = params(10)
    fac = orx.LFactors(orx.Model(10, 1e4 * G), 300.0)
    n = olay.ncoef(10)
    mat = np.zeros((3 * n, 3 * n), dtype=complex)
    for col in range(3 * n):
        e = np.zeros(3 * n, dtype=complex)
        e[col] = 1.0
        x = olay.unpack(e.reshape(-1, 3).T.copy(), 10)
        y = olay.pack(fac.apply(0.0, x))
        mat[:, col] = y.T.reshape(-1)
    lam = np.linalg.eigvals(mat)
    bad = -lam[np.argmax(np.abs(lam.imag))]
    with pytest.raises(SolverError):
        ShiftedLinearSolver(L, 300.0, p10).warm(np.array([bad]))


# ---------------------------------------------------------------- transforms

def test_transforms_t21_golden(golden_small):
    from paper_1805_06557_b200 import sphere as sp

    cfg = SphereConfig.for_truncation(21)
    st = unpack(golden_small["T21_sht_in"], 21)
    g = sp.synthesis(sp.SpectralField(st[0]), cfg).values
    assert rel_linf(g.ravel(), golden_small["T21_synth_phi"].ravel()) <= 1e-12
    u, v = sp.uv_from_vortdiv(sp.SpectralField(st[1]), sp.SpectralField(st[2]), cfg)
    assert rel_linf(u.values.ravel(), golden_small["T21_u"].ravel()) <= 1e-12
    assert rel_linf(v.values.ravel(), golden_small["T21_v"].ravel()) <= 1e-12
    an = sp.analysis(sp.GridField(golden_small["T21_grid_in"], cfg), cfg)
    assert rel_linf(pack(an.coeffs[None])[0], golden_small["T21_analysis"]) <= 1e-12


@pytest.mark.parametrize("atoms,key", [(1, "T21_tend_lc"), (2, "T21_tend_n"), (3, "T21_tend_lc_n")])
def test_tendencies_t21_golden(golden_small, atoms, key):
    cfg = SphereConfig.for_truncation(21)
    plan = plan_for(cfg)
    st = to_device(golden_small["T21_sht_in"])
    out = plan.tendency_dev(atoms, st).cpu().numpy()
    assert rel_linf(out, golden_small[key]) <= 1e-11


def test_tendency_t63_golden(golden_small):
    plan = plan_for(SphereConfig.for_truncation(63))
    out = plan.tendency_dev(3, to_device(golden_small["T63_sht_in"])).cpu().numpy()
    assert rel_linf(out, golden_small["T63_tend_lc_n"]) <= 1e-11


def test_tendency_t256_vs_oracle():
    g = osh.grid_for(256)
    st = ost.seeded_balanced_state(g)
    st[2] = ost.seeded_linear_state(256, 9)[2] * 1e-1  # give it divergence too
    ref = olay.pack(g.tendency_lc_n(st))
    plan = plan_for(SphereConfig.for_truncation(256))
    out = plan.tendency_dev(3, to_device(olay.pack(st))).cpu().numpy()
    assert rel_linf(out, ref) <= 1e-10


def test_sht_round_trip_t1279():
    """Size-independent property at cfg4's grid: analysis(synthesis(c)) = c."""
    cfg = SphereConfig.for_truncation(1279)
    plan = plan_for(cfg)
    c = ost.seeded_linear_state(1279, 5)[0:1] / 1e3
    cd = to_device(olay.pack(c))
    grid = plan.synthesis_dev(cd)
    back = plan.analysis_dev(grid).cpu().numpy()
    assert rel_linf(back, olay.pack(c)) <= 1e-10


# ---------------------------------------------------------------- ETD2RK

def test_etdrk_t42_golden(golden_medium):
    par = params(42)
    st = PrognosticState.from_stack(unpack(golden_medium["T42etd_ic"], 42), par.cfg)
    stepper = build_stepper("lg_rexi_lc_n_etdrk", par, RexiSetup(num_poles=128))
    s1 = stepper.step(st, 1800.0)
    assert rel_linf(pack(s1.stack()), golden_medium["T42etd_step1"]) <= 1e-10
    res = integrate(stepper, st, 1800.0, 8 * 1800.0)
    assert not res.diverged
    assert rel_l2(pack(res.state.stack()), golden_medium["T42etd_step8"]) <= 1e-8


def test_etdrk_t256_one_day_golden(golden_cfg2):
    """cfg2: 48 ETD2RK steps (1 simulated day) at T256, N=256, rel L2 <= 1e-8."""
    par = params(256)
    st = PrognosticState.from_stack(unpack(golden_cfg2["T256etd_ic"], 256), par.cfg)
    stepper = build_stepper("lg_rexi_lc_n_etdrk", par, RexiSetup(num_poles=256))
    s1 = stepper.step(st, 1800.0)
    assert rel_linf(pack(s1.stack()), golden_cfg2["T256etd_step1"]) <= 1e-10
    res = integrate(stepper, st, 1800.0, 48 * 1800.0)
    assert not res.diverged and res.n_steps == 48
    err = rel_l2(pack(res.state.stack()), golden_cfg2["T256etd_step48"])
    print(f"T256 one-day relative L2 vs reference: {err:.3e}")
    assert err <= 1e-8


# ---------------------------------------------------------------- cfg4 scale

def test_cfg4_t1279_subset_vs_oracle():
    """T1279 l-solve on 4 poles of the N=1024 contour vs the band-LU oracle,
    plus linearity of the full N=1024 pole sum."""
    trunc = 1279
    par = params(trunc)
    c = coeffs(1024)
    st = ost.seeded_linear_state(trunc, 0)
    sl = ShiftedLinearSolver(L, 14400.0, par)
    rhs = to_device(olay.pack(st))[None]
    bet = to_device(c.betas.reshape(1, -1))
    sub = sl.rexi_sum_dev(c.alphas, bet, rhs, pole_range=(0, 4), realify=False).cpu().numpy()[0]
    model = orx.Model(trunc, 1e4 * G)
    ref = olay.pack(orx.rexi_sum("l", model, 14400.0, c.alphas[:4], c.betas[:4], st, chunk=4,
                                 do_realify=False))
    assert rel_linf(sub, ref) <= LIN_BAR
    # linearity of the full sum: S(2x - y) = 2 S(x) - S(y) (up to rounding)
    st2 = ost.seeded_linear_state(trunc, 1)
    r2 = to_device(olay.pack(st2))[None]
    sx = sl.rexi_sum_dev(c.alphas, bet, rhs).cpu().numpy()
    sy = sl.rexi_sum_dev(c.alphas, bet, r2).cpu().numpy()
    sxy = sl.rexi_sum_dev(c.alphas, bet, (2.0 * rhs - r2).contiguous()).cpu().numpy()
    assert np.all(np.isfinite(sx))
    scale = np.max(np.abs(c.betas)) * 1e3
    assert np.max(np.abs(sxy - (2 * sx - sy))) <= 1e-10 * scale


def test_polecomm_nccl_single_rank_matches_serial():
    """The multi-rank reduce (NCCL all-gather + device tree combine, and the
    fast all-reduce variant) on a 1-rank group equals the serial sum."""
    import os
    import socket

    import torch.distributed as dist

    from paper_1805_06557_b200.parallel import PoleComm, distribute_terms, parallel_rexi_apply

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        par = params(42)
        c = coeffs(128)
        st = PrognosticState.from_stack(ost.seeded_linear_state(42, 7), par.cfg)
        for group in (LG, L):
            serial = rexi_step(group, st, 3600.0, c, par).stack()
            plan = distribute_terms(c.num_terms, 1)
            for det in (True, False):
                out, bd = parallel_rexi_apply(group, st, 3600.0, c, plan, par, comm=PoleComm(),
                                              deterministic=det)
                if det:
                    assert np.array_equal(out.stack(), serial)
                else:
                    assert rel_linf(pack(out.stack()), pack(serial)) <= 1e-13
                bd.validate()
    finally:
        dist.destroy_process_group()


def test_prepared_sum_bitwise_equals_unprepared():
    """swx_rexi_sum_prepared (cached lg factor tables) == swx_rexi_sum."""
    par = params(63)
    for group in (LG, L):
        sl = ShiftedLinearSolver(group, 3600.0, par)
        c0, c1 = coeffs(256, 0), coeffs(256, 1)
        rhs = to_device(np.stack([pack(ost.seeded_linear_state(63, 1)),
                                  pack(ost.seeded_linear_state(63, 2))]))
        bet = to_device(np.stack([c0.betas, c1.betas]))
        ref = sl.rexi_sum_dev(c0.alphas, bet, rhs).cpu().numpy()
        prep = sl.prepare_dev(c0.alphas, bet)
        out = torch.empty_like(rhs)
        got = sl.rexi_sum_prepared_dev(c0.alphas, bet, prep, rhs, out).cpu().numpy()
        assert np.array_equal(got, ref), group.token


@pytest.mark.parametrize("n_poles", [256, 1024])
def test_fused_axpy_sum_bitwise(n_poles):
    """swx_rexi_sum_prepared_axpy == prepared sum followed by swx_state_axpy,
    bitwise, for the single-chunk and the chunked (tree-combined) lg path and
    the Coriolis chain path."""
    from paper_1805_06557_b200.steppers import axpy
    par = params(63)
    for group in (LG, L):
        sl = ShiftedLinearSolver(group, 3600.0, par)
        c0 = coeffs(n_poles, 1)
        rhs = to_device(pack(ost.seeded_linear_state(63, 4))[None])
        base = to_device(pack(ost.seeded_linear_state(63, 5))[None])
        bet = to_device(c0.betas[None])
        prep = sl.prepare_dev(c0.alphas, bet)
        plain = sl.rexi_sum_prepared_dev(c0.alphas, bet, prep, rhs, torch.empty_like(rhs))
        ref = axpy(63, base, 1800.0, plain, torch.empty_like(rhs)).cpu().numpy()
        got = sl.rexi_sum_prepared_dev(c0.alphas, bet, prep, rhs, torch.empty_like(rhs),
                                       base=base, scale=1800.0).cpu().numpy()
        assert np.array_equal(got, ref), (group.token, n_poles)


def test_tendency_sub_bitwise():
    """swx_sht_tendency_sub == tendency followed by axpy(-1), bitwise (T63:
    fused table path; the plain difference is exercised by the T256 day)."""
    from paper_1805_06557_b200.steppers import axpy
    plan = plan_for(SphereConfig.for_truncation(63))
    g = osh.grid_for(63)
    st = to_device(olay.pack(ost.seeded_balanced_state(g)))
    sub = to_device(pack(ost.seeded_linear_state(63, 6)))
    t = plan.tendency_dev(3, st)
    ref = axpy(63, t, -1.0, sub, torch.empty_like(t)).cpu().numpy()
    got = plan.tendency_dev(3, st, sub=sub).cpu().numpy()
    assert np.array_equal(got, ref)


def test_stiffness_corner_chunked_poles_vs_oracle():
    """cfg3 corner (Phibar = 18000 g, dt = 3600 s, contour p1 = 80, N = 2048)
    at T85: the lg pole sum runs in 4 aligned chunks of 512 combined by the
    tree; two ETD2RK steps vs the oracle (rel L2 <= 1e-10)."""
    from paper_1805_06557_b200.workloads import seeded_balanced_state

    trunc, phibar, dt = 85, 18000.0 * G, 3600.0
    cfg = SphereConfig.for_truncation(trunc)
    par = ModelParams(phibar, cfg)
    grid = osh.Grid(trunc)
    ic = ost.seeded_balanced_state(grid)
    model = orx.Model(trunc, phibar)
    sets = {k: ost.contour_coeffs(k, 10.0, 80.0, 2048) for k in (0, 1, 2)}
    ref = ic
    for _ in range(2):
        ref = ost.etdrk2_step(model, grid, dt, sets, ref)
    stepper = build_stepper("lg_rexi_lc_n_etdrk", par, RexiSetup(10.0, 80.0, 2048))
    st = PrognosticState.from_stack(ic, cfg)
    for _ in range(2):
        st = stepper.step(st, dt)
    assert rel_l2(pack(st.stack()), olay.pack(ref)) <= 1e-10


@pytest.mark.parametrize("sid", ["lg_rexi_lc_n_erk_ver1", "lg_irk_lc_n_erk_ver0", "ln_erk"])
def test_split_and_explicit_steppers_golden(golden_split, sid):
    """Strang split ERK2 + REXI / Crank-Nicolson and fully explicit steppers
     against the reference, 2 steps at T21."""
    par = params(21)
    st = PrognosticState.from_stack(unpack(golden_split["T21split_ic"], 21), par.cfg)
    stepper = build_stepper(sid, par, RexiSetup(num_poles=64))
    for _ in range(2):
        st = stepper.step(st, 600.0)
    assert rel_l2(pack(st.stack()), golden_split[f"T21split_{sid}"]) <= 1e-10


@pytest.mark.parametrize("sid", ["lg_rexi_lc_n_erk_ver0", "lg_irk_lc_n_erk_ver1",
                                 "lg_rexi_lc_n_erk_ver1"])
def test_split_steppers_device_resident_match_host_path(sid):
    """The device-resident Strang split (one upload, three device sub-steps,
    one download) equals the host-composed path (taken when instrumented)
    to rounding, at T85."""
    import time

    from paper_1805_06557_b200.steppers import TimingCollector

    par = params(85)
    st0 = PrognosticState.from_stack(ost.seeded_balanced_state(osh.grid_for(85)), par.cfg)
    dev = build_stepper(sid, par, RexiSetup(num_poles=128))
    host = build_stepper(sid, par, RexiSetup(num_poles=128)).instrument(TimingCollector())
    a = dev.step(st0, 600.0)
    b = host.step(st0, 600.0)
    assert rel_l2(pack(a.stack()), pack(b.stack())) <= 1e-12
    for _ in range(3):  # warm both paths (plans, solvers, staging)
        dev.step(st0, 600.0)
        host.step(st0, 600.0)
    t0 = time.perf_counter()
    for _ in range(5):
        dev.step(st0, 600.0)
    t1 = time.perf_counter()
    for _ in range(5):
        host.step(st0, 600.0)
    t2 = time.perf_counter()
    print(f"{sid}: device-resident {(t1 - t0) / 5 * 1e3:.2f} ms, host-composed "
          f"{(t2 - t1) / 5 * 1e3:.2f} ms per step")


# ---------------------------------------------------------------- f4: IC, error, winds

@pytest.mark.parametrize("trunc", [21, 42])
def test_vortdiv_from_uv_golden(golden_io, trunc):
    """swx_sht_vortdiv vs the reference's vortdiv_from_uv (sphere.py:405-430)."""
    from paper_1805_06557_b200.sphere import GridField, vortdiv_from_uv

    cfg = SphereConfig.for_truncation(trunc)
    z, d = vortdiv_from_uv(GridField(golden_io[f"T{trunc}_u"], cfg),
                           GridField(golden_io[f"T{trunc}_v"], cfg), cfg)
    assert rel_linf(pack(z.coeffs), golden_io[f"T{trunc}_vort"]) <= 1e-11
    assert rel_linf(pack(d.coeffs), golden_io[f"T{trunc}_div"]) <= 1e-11


def test_galewsky_initial_state_and_error_golden(golden_io):
    """Balanced jet + bump at T42 (benchmarks.py:147-215) and the L-inf metric
    (benchmarks.py:290-306) vs the reference."""
    from paper_1805_06557_b200.benchmarks import init_barotropic_instability, linf_error

    cfg = SphereConfig.for_truncation(42)
    st = init_barotropic_instability(cfg, with_bump=True)
    st0 = init_barotropic_instability(cfg, with_bump=False)
    ref = golden_io["T42_galewsky"]
    for f in range(3):
        if np.abs(ref[f]).max() == 0:
            assert np.abs(pack(st.stack())[f]).max() == 0
        else:
            assert rel_linf(pack(st.stack())[f], ref[f]) <= 1e-10, f
    assert rel_linf(pack(st0.stack())[0], golden_io["T42_galewsky_nobump"][0]) <= 1e-10
    h = linf_error(st, st0, "h")
    assert abs(h - float(golden_io["T42_linf_h"])) <= 1e-9 * float(golden_io["T42_linf_h"])
    assert linf_error(st, st0, "vort") == 0.0


# ------------------------------------------------- column shards (§8f f1)

def _virtual_tendency(trunc, K, st, sub=None):
    """K co-resident column shards of one device run the sharded tendency in
    lockstep (virtual all-to-all); returns the assembled packed result."""
    from paper_1805_06557_b200.parallel import (ColumnShard, ShardedTendency, run_lockstep,
                                                virtual_exchange)
    cfg = SphereConfig.for_truncation(trunc)
    plan = plan_for(cfg)
    shards = [ColumnShard(cfg, r, K) for r in range(K)]
    tends = [ShardedTendency(plan, sh, 3) for sh in shards]
    outs = [torch.full_like(st, float("nan")) for _ in range(K)]
    run_lockstep((t.phases(st, o, sub) for t, o in zip(tends, outs)),
                 lambda items: virtual_exchange([t for t, _ in items], items[0][1]))
    full = torch.full_like(st, float("nan"))
    for sh, o in zip(shards, outs):
        a, b = sh.slots()
        full[:, a:b] = o[:, a:b]
    return full.cpu().numpy()


@pytest.mark.parametrize("trunc,ks", [(63, (1, 2, 3, 8)), (256, (2, 4, 8))])
def test_column_sharded_tendency_bitwise(trunc, ks):
    """m-sharded synthesis / latitude-sharded grid stage / m-sharded analysis
    with two all-to-alls == the single-rank fused tendency, bitwise."""
    g = osh.grid_for(trunc)
    st = ost.seeded_balanced_state(g)
    st[2] = ost.seeded_linear_state(trunc, 9)[2] * 1e-1
    oracle = olay.pack(g.tendency_lc_n(st))  # swe.py:188-279 restated on the CPU
    st = to_device(olay.pack(st))
    sub_h = pack(ost.seeded_linear_state(trunc, 6))
    sub = to_device(sub_h)
    plan = plan_for(SphereConfig.for_truncation(trunc))
    ref = plan.tendency_dev(3, st).cpu().numpy()
    ref_sub = plan.tendency_dev(3, st, sub=sub).cpu().numpy()
    for K in ks:
        got = _virtual_tendency(trunc, K, st)
        assert np.array_equal(got, ref), K
        assert rel_linf(got, oracle) <= 1e-10, K            # the shards against the oracle itself
        got = _virtual_tendency(trunc, K, st, sub)
        assert np.array_equal(got, ref_sub), K
        assert rel_linf(got, oracle - sub_h) <= 1e-10, K


def test_column_sharded_etdrk_bitwise():
    """cfg2-shaped ETD2RK (T85, N=128) on 3 column shards: lg pole sums on the
    own columns, sharded tendencies; 2 steps == the single-rank engine."""
    from paper_1805_06557_b200.parallel import (ColumnEtdrkEngine, ColumnShard, run_lockstep,
                                                virtual_exchange)
    from paper_1805_06557_b200.steppers import EtdrkStepper
    trunc, K, dt = 85, 3, 1800.0
    par = params(trunc)
    ic = ost.seeded_balanced_state(osh.grid_for(trunc))
    stepper = EtdrkStepper(LG, LC_N, par, RexiSetup(num_poles=128))
    sets = stepper.coeff_set(dt)
    ref = stepper.engine(dt)
    ref.load(ic)
    engines = [ColumnEtdrkEngine(LG, LC_N, par, dt, sets, ColumnShard(par.cfg, r, K))
               for r in range(K)]
    for e in engines:
        e.load(ic)
    for _ in range(2):
        ref.step_dev()
        run_lockstep((e.phases() for e in engines),
                     lambda items: virtual_exchange([t for t, _ in items], items[0][1]))
    want = ref.u.cpu().numpy()
    # the same two steps by the CPU oracle (steppers.py:238-269 restated)
    grid = osh.grid_for(trunc)
    osets = {k: (np.asarray(sets[k].alphas), np.asarray(sets[k].betas)) for k in (0, 1, 2)}
    model = orx.Model(trunc, 1e4 * G)
    oref = ic
    for _ in range(2):
        oref = ost.etdrk2_step(model, grid, dt, osets, oref)
    oref = olay.pack(oref)
    for e in engines:
        a, b = e.shard.slots()
        own = e.own().cpu().numpy()
        assert np.array_equal(own, want[:, a:b]), e.shard.rank
        assert rel_l2(own, oref[:, a:b]) <= 1e-9, e.shard.rank


def test_lg_column_restricted_sum_bitwise():
    """swx_solver_set_columns: the own columns of a restricted lg pole sum
    equal the full sum bitwise; the Coriolis group refuses column shards."""
    from paper_1805_06557_b200.errors import ConfigurationError
    par = params(63)
    c = coeffs(128)
    st = to_device(pack(ost.seeded_linear_state(63, 2)))[None]
    b = to_device(np.asarray(c.betas).reshape(1, -1))
    full = ShiftedLinearSolver(LG, 900.0, par).rexi_sum_dev(c.alphas, b, st).cpu().numpy()
    from paper_1805_06557_b200.parallel import column_slots
    for m0, m1 in ((0, 9), (9, 40), (40, 64), (63, 64)):
        s = ShiftedLinearSolver(LG, 900.0, par, columns=(m0, m1))
        got = s.rexi_sum_dev(c.alphas, b, st).cpu().numpy()
        a, z = column_slots(63, m0, m1)
        assert np.array_equal(got[..., a:z], full[..., a:z]), (m0, m1)
    with pytest.raises(ConfigurationError):
        ShiftedLinearSolver(L, 900.0, par, columns=(0, 9)).warm(c.alphas)


@pytest.mark.parametrize("K", [2, 3])
def test_column_sharded_t1279_round_trip(K):
    """cfg4's SH round trip on K column/latitude shards (virtual ranks in
    lockstep): every rank's grid rows and coefficient columns equal the
    single-rank transforms (the Legendre sums bitwise; longitude FFTs over
    row subsets within 1e-15), and the round trip returns the field."""
    from paper_1805_06557_b200.parallel import (ColumnShard, ShardedTransforms, run_lockstep,
                                                virtual_exchange)
    cfg = SphereConfig.for_truncation(1279)
    plan = plan_for(cfg)
    c = to_device(olay.pack(ost.seeded_linear_state(1279, 5)[0:1] / 1e3))
    ref_grid = plan.synthesis_dev(c)
    ref_back = plan.analysis_dev(ref_grid)
    xs = [ShardedTransforms(plan, ColumnShard(cfg, r, K)) for r in range(K)]
    grids = [torch.full_like(ref_grid, float("nan")) for _ in range(K)]
    backs = [torch.full_like(ref_back, float("nan")) for _ in range(K)]
    ex = lambda items: virtual_exchange([t for t, _ in items], items[0][1])  # noqa: E731
    run_lockstep((x.synthesis_phases(c, g) for x, g in zip(xs, grids)), ex)
    full = torch.full_like(ref_grid, float("nan"))
    for x, g in zip(xs, grids):
        rows = torch.as_tensor(x.own_rows(), device=g.device)
        full[:, rows] = g[:, rows]
    scale = ref_grid.abs().max()
    assert float((full - ref_grid).abs().max() / scale) <= 1e-15
    run_lockstep((x.analysis_phases(full, b) for x, b in zip(xs, backs)), ex)
    got = torch.full_like(ref_back, float("nan"))
    for x, b in zip(xs, backs):
        a, z = x.shard.slots()
        got[:, a:z] = b[:, a:z]
    assert float((got - ref_back).abs().max() / ref_back.abs().max()) <= 1e-14
    assert rel_linf(got.cpu().numpy(), c.cpu().numpy()) <= 1e-10


def test_cfg3_stiffness_sweep_t256_matches_oracle_verdicts():
    """cfg3: all 36 (Phibar, dt) cases of the stiffness sweep at T256
    (contours per workloads.stiffness_cases, N up to 2048), 24 device-resident
    ETD2RK steps each with the reference's blow-up check (synthesis of phi',
    |phi'| > 1e6, steppers.py:516-520) after every step.  Cases the oracle
    integrated (tests/golden/cfg3_verdicts.json) must blow up at the same step
    (or stay stable); every other case must stay stable."""
    import json
    import os
    from paper_1805_06557_b200.steppers import EtdrkStepper
    from paper_1805_06557_b200.workloads import seeded_balanced_state, stiffness_cases
    with open(os.path.join(os.path.dirname(__file__), "golden", "cfg3_verdicts.json")) as fh:
        verdicts = json.load(fh)
    cfg = SphereConfig.for_truncation(256)
    plan = plan_for(cfg)
    ic = seeded_balanced_state(cfg)
    cases = stiffness_cases()
    assert len(cases) == 36 and max(c.y for c in cases) < 61.0
    for case in cases:
        par = ModelParams(case.phibar, cfg)
        eng = EtdrkStepper(LG, LC_N, par, RexiSetup(10.0, case.p1, case.n_poles)).engine(case.dt)
        eng.load(ic)
        blow = None
        for k in range(1, case.steps + 1):
            eng.step_dev()
            phi = plan.synthesis_dev(eng.u[0:1].contiguous())
            if not bool(torch.isfinite(phi).all()) or float(phi.abs().max()) > 1e6:
                blow = k
                break
        want = verdicts.get(f"{case.phibar_g:.0f},{case.dt:.0f}", {"blow_up_step": None})
        assert blow == want["blow_up_step"], (case, blow, want)


def test_cfg3_mid_case_24_steps_vs_oracle():
    """A mid cfg3 case (Phibar = 10000 g, dt = 1800 s: p1 = 30, N = 256) for the
    full 24 steps at T85 against the oracle trajectory (rel L2 <= 1e-8)."""
    from paper_1805_06557_b200.workloads import stiffness_cases
    case = next(c for c in stiffness_cases() if c.phibar_g == 10000 and c.dt == 1800.0)
    trunc = 85
    cfg = SphereConfig.for_truncation(trunc)
    par = ModelParams(case.phibar, cfg)
    grid = osh.Grid(trunc)
    ic = ost.seeded_balanced_state(grid)
    model = orx.Model(trunc, case.phibar)
    sets = {k: ost.contour_coeffs(k, 10.0, case.p1, case.n_poles) for k in (0, 1, 2)}
    ref = ic
    for _ in range(case.steps):
        ref = ost.etdrk2_step(model, grid, case.dt, sets, ref)
    stepper = build_stepper("lg_rexi_lc_n_etdrk", par, RexiSetup(10.0, case.p1, case.n_poles))
    res = integrate(stepper, PrognosticState.from_stack(ic, cfg), case.dt, case.steps * case.dt)
    assert not res.diverged
    assert rel_l2(pack(res.state.stack()), olay.pack(ref)) <= 1e-8


@pytest.mark.parametrize("trunc", [42, 85])
def test_table_free_transforms_and_tendency_vs_oracle(trunc, monkeypatch):
    """The on-the-fly (table-free) paths that serve T > ~340 -- column-walk
    plain analysis, state synthesis + cuFFT grid stage + column-walk tendency
    analysis (with the fused subtraction) -- forced at small T
    (SWX_SHT_TABLE=0) against the oracle."""
    from paper_1805_06557_b200.sphere import ShtPlan
    monkeypatch.setenv("SWX_SHT_TABLE", "0")
    cfg = SphereConfig.for_truncation(trunc)
    plan = ShtPlan(cfg)
    assert not plan.fused_stages()
    g = osh.grid_for(trunc)
    st = ost.seeded_balanced_state(g)
    st[2] = ost.seeded_linear_state(trunc, 9)[2] * 1e-1
    ref = olay.pack(g.tendency_lc_n(st))
    dst = to_device(olay.pack(st))
    out = plan.tendency_dev(3, dst).cpu().numpy()
    assert rel_linf(out, ref) <= 1e-10
    sub = to_device(pack(ost.seeded_linear_state(trunc, 6)))
    got = plan.tendency_dev(3, dst, sub=sub).cpu().numpy()
    assert rel_linf(got, ref - sub.cpu().numpy()) <= 1e-10
    c = ost.seeded_linear_state(trunc, 5)[0:1] / 1e3
    back = plan.analysis_dev(plan.synthesis_dev(to_device(olay.pack(c)))).cpu().numpy()
    assert rel_linf(back, olay.pack(c)) <= 1e-10


def test_etdrk_graph_capture_above_fused_range():
    """T > 341 (cuFFT grid stage, no fused stages): the ETD2RK step graph
    captures (psi0 waits on the synthesis event of the non-fused path too) and
    equals the uncaptured engine bitwise over two steps."""
    from paper_1805_06557_b200.steppers import EtdrkStepper
    from paper_1805_06557_b200.workloads import seeded_balanced_state
    trunc = 383
    par = params(trunc)
    ic = seeded_balanced_state(par.cfg)
    outs = []
    for graph in (True, False):
        eng = EtdrkStepper(LG, LC_N, par, RexiSetup(num_poles=128), graph=graph).engine(900.0)
        assert not eng.plan.fused_stages()
        eng.load(ic)
        for _ in range(2):
            eng.step_dev()
        outs.append(eng.u.cpu().numpy())
    assert np.all(np.isfinite(outs[0])) and np.array_equal(outs[0], outs[1])


def test_t1279_tendency_table_vs_column_walk(monkeypatch):
    """At T1279 the tendency analysis streams the 6.3 GB parity-split Legendre table
    (TMA + DMMA); the table-free column walk (validated against the oracle
    at small T) gives the same tendency to rounding."""
    from paper_1805_06557_b200.sphere import ShtPlan
    from paper_1805_06557_b200.workloads import seeded_balanced_state
    cfg = SphereConfig.for_truncation(1279)
    st = to_device(pack(seeded_balanced_state(cfg)))
    a = plan_for(cfg).tendency_dev(3, st)
    monkeypatch.setenv("SWX_SHT_TABLE", "0")
    b = ShtPlan(cfg).tendency_dev(3, st)
    assert float((a - b).abs().max() / b.abs().max()) <= 1e-12


def test_integration_md_binding_example(golden_small):
    """The ctypes binding INTEGRATION.md shows a swerexi maintainer (section 2)
    runs as written against the library and reproduces the reference's cfg0
    lg REXI step."""
    import os
    import re
    from paper_1805_06557_b200 import _lib as L
    from paper_1805_06557_b200.rexi import RexiSetup
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(root, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# swerexi/gpu_solver\.py.*?)```", text, re.S).group(1)
    code = code.replace('ctypes.CDLL("libswx.so")', f'ctypes.CDLL({L.LIB_PATH!r})')
    ns = {"SolverError": RuntimeError}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    par = params(63)
    coeffs = RexiSetup().coefficients("psi0", 3600.0)
    solver = ns["GpuShiftedSolver"]("lg", 3600.0, par)
    out = solver.rexi_sum(coeffs.alphas, coeffs.betas, unpack(golden_small["cfg0_in"], 63))
    assert rel_linf(out, golden_small["cfg0_out"]) <= LIN_BAR


@pytest.mark.parametrize("K", [2, 3])
def test_column_sharded_tendency_direct_push_bitwise(K):
    """The peer-memory exchange (swx_sht_shard_push: each rank copies its
    blocks straight into the peers' workspaces, no slabs, no all-to-all) with
    co-resident virtual ranks: bitwise equal to the single-rank tendency."""
    from paper_1805_06557_b200.parallel import (ColumnShard, ShardedTendency, run_lockstep,
                                                virtual_push)
    trunc = 256
    cfg = SphereConfig.for_truncation(trunc)
    plan = plan_for(cfg)
    g = osh.grid_for(trunc)
    st = ost.seeded_balanced_state(g)
    st[2] = ost.seeded_linear_state(trunc, 9)[2] * 1e-1
    st = to_device(olay.pack(st))
    ref = plan.tendency_dev(3, st).cpu().numpy()
    shards = [ColumnShard(cfg, r, K) for r in range(K)]
    tends = [ShardedTendency(plan, sh, 3) for sh in shards]
    for t in tends:
        t.direct = True
    outs = [torch.full_like(st, float("nan")) for _ in range(K)]
    run_lockstep((t.phases(st, o) for t, o in zip(tends, outs)),
                 lambda items: virtual_push([t for t, _ in items], items[0][1]))
    full = np.full(ref.shape, np.nan, dtype=ref.dtype)
    for sh, o in zip(shards, outs):
        a, b = sh.slots()
        full[:, a:b] = o[:, a:b].cpu().numpy()
    assert np.array_equal(full, ref)


@pytest.mark.parametrize("trunc,K", [(63, 3), (85, 2), (256, 2), (256, 4)])
def test_column_sharded_tendency_peer_stores_bitwise(trunc, K):
    """Fused exchange: the synthesis and grid-stage epilogues store straight
    into the owners' workspaces (virtual ranks' workspaces on one GPU stand in
    for peer-mapped memory); no copies, only the stage ordering.  Bitwise
    equal to the single-rank tendency (with and without the subtraction)."""
    from paper_1805_06557_b200.parallel import ColumnShard, ShardedTendency, run_lockstep
    cfg = SphereConfig.for_truncation(trunc)
    plan = plan_for(cfg)
    g = osh.grid_for(trunc)
    st = ost.seeded_balanced_state(g)
    st[2] = ost.seeded_linear_state(trunc, 9)[2] * 1e-1
    st = to_device(olay.pack(st))
    sub = to_device(pack(ost.seeded_linear_state(trunc, 6)))
    for sb in (None, sub):
        ref = plan.tendency_dev(3, st, sub=sb).cpu().numpy()
        shards = [ColumnShard(cfg, r, K) for r in range(K)]
        tends = [ShardedTendency(plan, sh, 3) for sh in shards]
        addrs = [t.workspace.data_ptr() for t in tends]
        for t in tends:
            t.use_peer_stores(addrs)
        outs = [torch.full_like(st, float("nan")) for _ in range(K)]
        run_lockstep((t.phases(st, o, sb) for t, o in zip(tends, outs)), lambda items: None)
        full = np.full(ref.shape, np.nan, dtype=ref.dtype)
        for sh, o in zip(shards, outs):
            a, b = sh.slots()
            full[:, a:b] = o[:, a:b].cpu().numpy()
        assert np.array_equal(full, ref), (trunc, K, sb is None)


def test_l_rexi_n_etdrk_vs_oracle():
    """The paper's ETD2RK with the full linear operator L = L_g + L_c by REXI
    (Coriolis chain solves with the fused ETD2RK epilogues) and N alone as the
    remainder (build_stepper("l_rexi_n_etdrk")), 3 steps at T42 vs the oracle."""
    from oracle import stepping as ostep
    trunc, dt, n = 42, 1200.0, 128
    par = params(trunc)
    grid = osh.Grid(trunc)
    ic = ost.seeded_balanced_state(grid)
    model = orx.Model(trunc, 1e4 * G)
    sets = {k: ost.contour_coeffs(k, 10.0, 30.0, n) for k in (0, 1, 2)}
    fac = orx.LFactors(model, dt)
    ref = ic
    for _ in range(3):
        ref = ostep.etdrk2_step(model, grid, dt, sets, ref, group="l", remainder="n", factors=fac)
    stepper = build_stepper("l_rexi_n_etdrk", par, RexiSetup(10.0, 30.0, n))
    res = integrate(stepper, PrognosticState.from_stack(ic, par.cfg), dt, 3 * dt)
    assert not res.diverged
    assert rel_l2(pack(res.state.stack()), olay.pack(ref)) <= 1e-10


@pytest.mark.parametrize("trunc", [170, 300, 341])
def test_fused_stockham_grid_stage_vs_table_free(trunc, monkeypatch):
    """Truncations whose tendency FFT length has no register-FFT split
    (Stockham fused grid stage, nlon_t up to 1024) agree with the table-free
    path (cuFFT grid stage + column-walk analysis) to rounding."""
    from paper_1805_06557_b200.sphere import ShtPlan
    from paper_1805_06557_b200.workloads import seeded_balanced_state
    cfg = SphereConfig.for_truncation(trunc)
    plan = plan_for(cfg)
    assert plan.fused_stages()
    st = seeded_balanced_state(cfg)
    st[2] = ost.seeded_linear_state(trunc, 9)[2] * 1e-1
    st = to_device(pack(st))
    a = plan.tendency_dev(3, st)
    monkeypatch.setenv("SWX_SHT_TABLE", "0")
    b = ShtPlan(cfg).tendency_dev(3, st)
    assert float((a - b).abs().max() / b.abs().max()) <= 1e-12


def test_cfg4_pole_blocks_combine_bitwise():
    """cfg4 at full size (T1279, N = 1024, pivot-cached chains): the per-rank
    partials of K = 2 and 8 contiguous pole blocks, combined by the fixed tree,
    equal the one-launch sum bitwise (the multi-GPU decomposition's
    determinism at the size it is meant for)."""
    trunc = 1279
    par = params(trunc)
    c = coeffs(1024)
    sl = ShiftedLinearSolver(L, 14400.0, par)
    rhs = to_device(olay.pack(ost.seeded_linear_state(trunc, 0)))[None]
    bet = to_device(c.betas.reshape(1, -1))
    full = sl.rexi_sum_dev(c.alphas, bet, rhs).cpu().numpy()
    lib = _lib.load()
    for k in (2, 8):
        parts = torch.stack([sl.rexi_sum_dev(c.alphas, bet, rhs,
                                             pole_range=(r * 1024 // k, (r + 1) * 1024 // k),
                                             realify=False) for r in range(k)]).contiguous()
        out = torch.empty_like(rhs)
        _lib.check(lib.swx_tree_combine(trunc, 1, k, ptr(parts), 1, ptr(out), stream_ptr()))
        assert np.array_equal(out.cpu().numpy(), full), k


def test_l_group_without_rotation_equals_lg():
    """With Omega = 0 the Coriolis chains decouple: the l pole sum equals the
    lg one (test_solvers.py:86-98 analogue, 1e-13)."""
    par = params(42, omega=0.0)
    c = coeffs(128)
    st = ost.seeded_linear_state(42, 3)
    a = ShiftedLinearSolver(L, 1800.0, par).rexi_sum(c.alphas, c.betas, st)
    b = ShiftedLinearSolver(LG, 1800.0, par).rexi_sum(c.alphas, c.betas, st)
    assert rel_linf(pack(a), pack(b)) <= 1e-13


def test_gravity_eigenmode_rexi_step():
    """REXI on a gravity eigenmode of one (l, m) returns e^{i omega dt} times
    the mode (test_steppers.py:208-213 analogue, 1e-10): L_g on (phi', div)
    is [[0, -Phibar], [kappa_l, 0]] (swe.py:169-185)."""
    trunc, l, m, dt = 42, 9, 3, 900.0
    par = params(trunc)
    phibar = par.mean_geopotential
    kap = l * (l + 1) / par.cfg.radius_a ** 2
    omega = np.sqrt(phibar * kap)
    st = np.zeros((3, trunc + 1, trunc + 1), dtype=np.complex128)
    st[0, l, m] = phibar       # eigenvector (phi', div) = (Phibar, -i omega) for lambda = i omega
    st[2, l, m] = -1j * omega
    c = RexiSetup().coefficients("psi0", dt)
    out = ShiftedLinearSolver(LG, dt, par).rexi_sum(c.alphas, c.betas, st)
    want = st * np.exp(1j * omega * dt)
    assert np.max(np.abs(out - want)) <= 1e-10 * np.max(np.abs(want))


def test_captured_graph_survives_shift_set_eviction(golden_medium):
    """A captured ETD2RK graph keeps its shift set alive when more than
    _MAX_SETS other sets pass through the shared get_solver instance."""
    from paper_1805_06557_b200.solvers import ShiftedLinearSolver, get_solver

    par = params(42)
    st = PrognosticState.from_stack(unpack(golden_medium["T42etd_ic"], 42), par.cfg)
    stepper = build_stepper("lg_rexi_lc_n_etdrk", par, RexiSetup(num_poles=128))
    s1 = pack(stepper.step(st, 1800.0).stack())  # captures the step graph
    sol = get_solver("lg", 1800.0, par)
    for k in range(ShiftedLinearSolver._MAX_SETS + 2):
        sol.warm(coeffs(16 + 4 * k).alphas)
        torch.zeros(1 << 22, dtype=torch.complex128, device="cuda")  # churn the allocator
    again = pack(stepper.step(st, 1800.0).stack())
    assert np.array_equal(again, s1)
    assert rel_linf(again, golden_medium["T42etd_step1"]) <= 1e-10


def test_instrumented_etdrk_step_fills_breakdown(golden_medium):
    """instrument(collector): the reference's instrumented ETD2RK path
    (steppers.py:416-443) -- psi_k through parallel_rexi_apply, timed
    tendencies -- fills every category and gives the same step."""
    from paper_1805_06557_b200.steppers import TimingCollector

    par = params(42)
    st = PrognosticState.from_stack(unpack(golden_medium["T42etd_ic"], 42), par.cfg)
    stepper = build_stepper("lg_rexi_lc_n_etdrk", par, RexiSetup(num_poles=128))
    col = TimingCollector()
    stepper.instrument(col, workers=2)
    s1 = pack(stepper.step(st, 1800.0).stack())
    assert rel_linf(s1, golden_medium["T42etd_step1"]) <= 1e-10
    for name in ("overall", "nonlinearities", "rexi_total", "broadcast", "term_solves", "reduce"):
        assert getattr(col, name) > 0.0, name
    assert col.nonlinearities < col.overall


# ------------------------------------------------ partition form of the l chains

@pytest.mark.parametrize("trunc,n_poles", [(1, 3), (2, 8), (7, 5), (8, 33), (16, 40), (33, 31),
                                           (64, 64), (65, 17), (129, 40), (200, 12), (255, 40)])
def test_l_partition_kernel_edge_truncations_vs_oracle(trunc, n_poles):
    """The warp-per-system partition solve (rexi_l_part_kernel, every T <= 255):
    every lanes-per-system class (columns of 1..256 rows: W = 1..32, q = 2..8),
    padded last lanes, pole counts that are not multiples of the 32-pole block
    or of the poles per pass, against the oracle's band LU (solvers.py:196-212)."""
    st = ost.seeded_linear_state(trunc, 5)
    a, b = ost.contour_coeffs(0, 10.0, 30.0, n_poles)
    model = orx.Model(trunc, 1e4 * G)
    ref = olay.pack(orx.rexi_sum("l", model, 1800.0, a, b, st))
    sl = ShiftedLinearSolver(L, 1800.0, params(trunc))
    out = sl.rexi_sum_dev(a, to_device(np.asarray(b).reshape(1, -1)), to_device(pack(st))[None])
    assert rel_linf(out[0].cpu().numpy(), ref) <= LIN_BAR


def test_l_partition_kernel_two_rhs_and_pole_subranges_t255():
    """T255 (the largest truncation the partition kernel serves: 32 lanes x 8
    rows): two fused right-hand sides against the oracle, and unaligned pole
    sub-ranges summing to the full result."""
    trunc, n = 255, 48
    par = params(trunc)
    sl = ShiftedLinearSolver(L, 900.0, par)
    c0, c1 = coeffs(n, 0), coeffs(n, 1)
    u, v = ost.seeded_linear_state(trunc, 1), ost.seeded_linear_state(trunc, 2)
    rhs = to_device(np.stack([pack(u), pack(v)]))
    bet = to_device(np.stack([c0.betas, c1.betas]))
    out = sl.rexi_sum_dev(c0.alphas, bet, rhs).cpu().numpy()
    model = orx.Model(trunc, 1e4 * G)
    for r, (st, c) in enumerate(((u, c0), (v, c1))):
        ref = olay.pack(orx.rexi_sum("l", model, 900.0, c.alphas, c.betas, st))
        assert rel_linf(out[r], ref) <= LIN_BAR
    parts = [sl.rexi_sum_dev(c0.alphas, bet, rhs, pole_range=pr, realify=False).cpu().numpy()
             for pr in ((0, 7), (7, 39), (39, 48))]
    tot = parts[0] + parts[1] + parts[2]
    unreal = sl.rexi_sum_dev(c0.alphas, bet, rhs, realify=False).cpu().numpy()
    assert rel_linf(tot[0], unreal[0]) <= 1e-12 and rel_linf(tot[1], unreal[1]) <= 1e-12
