"""Benchmark of the REXI hot path on B200 (driver contract).

Default workload = BASELINE.json config 2 (the metric is quoted at T256):
``lg_rexi_lc_n_etdrk`` at T256 (386 x 772 grid), N = 256 REXI poles,
dt = 1800 s, seeded balanced vorticity state (peak 1e-5 1/s).
A step = one ETD2RK step = 3 fused REXI pole sums (psi0+psi1 fused, psi2)
+ 2 fused LC+N tendencies.  Metric: REXI pole-solves x SH-coeffs per second
(3 * N * ncoef units per step) and wall time per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg0|cfg1|cfg2|cfg4]

N > 1 runs under torchrun: poles are sharded over ranks (strong scaling),
with one deterministic all-gather+tree reduce per REXI application.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=48)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=("cfg0", "cfg1", "cfg2", "cfg3", "cfg4", "etd1279"),
                    default="cfg2")
    ap.add_argument("--shard", choices=("auto", "poles", "cols", "cols-p2p", "cols-fused"),
                    default="auto",
                    help="N>1: shard REXI poles (+ all-reduce) or zonal columns (ETD2RK: "
                         "sharded N term, 4 all-to-alls per step; cols-p2p: direct copies "
                         "into the peers' symmetric-memory workspaces; cols-fused: the stage "
                         "kernels store into the peers' workspaces); auto = cols for cfg2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--profile", action="store_true",
                    help="ncu mode: only warm-up + the K timed steps (no soak/e2e/cpu/breakdown)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        self.gpu = gpu_index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- reference arm

def run_reference(args, rank, world):
    """The reference's CPU algorithm (the oracle port: the reference is a
    Python package and cannot travel to the GPU box) on the host cores, on
    our arm's workload; each step is one full step of that workload, the
    timed sample stops after K steps or 150 s, whichever comes first."""
    if rank != 0:
        return
    from oracle import layout as olay
    from oracle import rexi as orx
    from oracle import sht as osh
    from oracle import stepping as ost
    from paper_1805_06557_b200.workloads import CONFIGS

    w = CONFIGS[args.config]
    if w.trunc > 341 and w.stepper == "lg_rexi_lc_n_etdrk":
        print(json.dumps({"impl": "reference", "unavailable":
                          "the CPU transforms need dense Legendre tables of ~25 GB each at T1279"}))
        return
    model = orx.Model(w.trunc, w.phibar)
    nc = olay.ncoef(w.trunc)
    if w.stepper == "lg_rexi_lc_n_etdrk":
        grid = osh.grid_for(w.trunc)
        st = ost.seeded_balanced_state(grid)
        sets = {k: ost.contour_coeffs(k, w.p0, w.p1, w.n_poles) for k in (0, 1, 2)}
        step = lambda s: ost.etdrk2_step(model, grid, w.dt, sets, s)  # noqa: E731
        units = 3 * w.n_poles * nc
    else:
        st = ost.seeded_linear_state(w.trunc, 0)
        a, b = ost.contour_coeffs(0, w.p0, w.p1, w.n_poles)
        fac = orx.LFactors(model, w.dt) if w.group == "l" else None
        step = lambda s: orx.rexi_sum(w.group, model, w.dt, a, b, s, fac)  # noqa: E731
        units = w.n_poles * nc
    for _ in range(min(args.warmup, 1)):
        st = step(st)
    times = []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        st = step(st)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > 150.0:
            break
    sec = sum(times) / len(times)
    cores = len(os.sched_getaffinity(0))
    val = units / sec
    line = {
        "impl": "reference", "metric": "REXI pole-solves*SH-coeffs/s", "value": val,
        "unit": "pole-solve*coeff/s", "n_gpus": world, "steps": len(times),
        "steps_requested": args.steps, "warmup": min(args.warmup, 1), "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded, SURVEY §8d)",
        "config": bench_config(w),
        "cpu_baseline": {"value": val, "unit": "pole-solve*coeff/s", "cores": cores,
                         "kind": "port",
                         "sample": f"{len(times)} full steps of {w.name} (numpy/scipy oracle, "
                                   f"{cores} host threads for BLAS)" + PORT_NOTE},
        "e2e": {"value": val, "unit": "pole-solve*coeff/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


PORT_NOTE = ("; kind 'port': the oracle restatement of swerexi, measured 1.1-1.2x slower than swerexi itself on 8 cores of the build container (VERDICT r1), so ratios against it are that much generous")


def bench_config(w) -> dict:
    """The workload description both arms emit verbatim (same keys, same
    values), so the driver can match the two lines; per-arm details go to
    ``run_info``."""
    return {"workload": w.name, "trunc": w.trunc, "grid": [w.params.cfg.nlat, w.params.cfg.nlon],
            "n_poles": w.n_poles, "dt": w.dt,
            "l2": "GPU arm: flushed (256 MB write) before every timed step; CPU arm: n/a"}


# ---------------------------------------------------------------- our arm

def fp64_peak_tflops(torch, lib, _lib):
    n_blocks = torch.cuda.get_device_properties(0).multi_processor_count * 8
    sink = torch.empty(n_blocks * 256, dtype=torch.float64, device="cuda")
    iters = 4096
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        _lib.check(lib.swx_fp64_fma_probe(sink.data_ptr(), n_blocks, iters, s))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(5):
        e0.record()
        _lib.check(lib.swx_fp64_fma_probe(sink.data_ptr(), n_blocks, iters, s))
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = max(best, n_blocks * 256 * iters * 8 * 2 / (ms * 1e-3) / 1e12)
    return best


def _tendency_nlon(trunc: int, nlon: int) -> int:
    """The tendency FFT length libswx uses: smallest 7-smooth n >= 3T+1
    (the grid's nlon when already 7-smooth), see csrc/sht.cu."""
    def smooth(n):
        for f in (2, 3, 5, 7):
            while n % f == 0:
                n //= f
        return n == 1
    need = 3 * trunc + 1
    if nlon >= need and smooth(nlon):
        return nlon
    n = max(need, 2)
    n += n & 1
    while not smooth(n):
        n += 2
    return n


def _hbm_peak() -> float:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 7700.0  # B200_PROFILING.md fallback


def load_traffic():
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        try:
            with open(path) as fh:
                return json.load(fh)
        except Exception:
            return {}
    return {}


def _l_cache_bytes(dr):
    """Size of the warm-time pivot cache of an l solver (0: lg, or not built)."""
    from paper_1805_06557_b200 import _lib
    return int(_lib.load().swx_solver_cache_bytes(dr.solver._native(dr.alphas).h))


def run_stiffness(args, rank, world):
    """cfg3: config 2's ETD2RK setup over the 36-case stiffness sweep
    (workloads.stiffness_cases), 24 device-resident steps per case (graph
    replays, L2 flushed before each step, CUDA events around each step); the
    line's value is the sweep's total pole-solve*coeff over its total time,
    and every case must stay finite (the reference's blow-up check,
    steppers.py:516-520).  Replicated on every rank (the sweep's cases are
    independent; each rank runs the whole sweep) -- one GPU is the unit."""
    import torch

    from paper_1805_06557_b200.device import ncoef
    from paper_1805_06557_b200.rexi import RexiSetup
    from paper_1805_06557_b200.steppers import EtdrkStepper
    from paper_1805_06557_b200.swe import LC_N, LG, ModelParams
    from paper_1805_06557_b200.sphere import SphereConfig, plan_for
    from paper_1805_06557_b200.workloads import seeded_balanced_state, stiffness_cases

    cfg = SphereConfig.for_truncation(256)
    nc = ncoef(256)
    plan = plan_for(cfg)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    sampler = ClockSampler(0)
    sampler.start()
    rows, tot_units, tot_ms, stable = [], 0.0, 0.0, True
    ic = seeded_balanced_state(cfg)  # config 2's initial state for every case
    for case in stiffness_cases():
        par = ModelParams(case.phibar, cfg)
        eng = EtdrkStepper(LG, LC_N, par, RexiSetup(10.0, case.p1, case.n_poles)).engine(case.dt)
        eng.load(ic)
        for _ in range(max(1, args.warmup)):
            eng.step_dev()
        eng.load(ic)
        torch.cuda.synchronize()
        ms, blow = 0.0, None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for k in range(1, case.steps + 1):
            flush.zero_()
            e0.record()
            eng.step_dev()
            e1.record()
            e1.synchronize()
            ms += e0.elapsed_time(e1)
            if blow is None:  # the reference's blow-up check (untimed)
                phi = plan.synthesis_dev(eng.u[0:1].contiguous())
                if not bool(torch.isfinite(phi).all()) or float(phi.abs().max()) > 1e6:
                    blow = k
        ok = blow is None
        stable &= ok
        units = 3.0 * case.n_poles * nc * case.steps
        tot_units += units
        tot_ms += ms
        rows.append({"phibar_g": case.phibar_g, "dt": case.dt, "y": round(case.y, 2),
                     "p1": case.p1, "n_poles": case.n_poles,
                     "ms_per_step": round(ms / case.steps, 4), "stable": ok,
                     "blow_up_step": blow})
    clocks = sampler.stop()
    line = {"metric": "REXI pole-solves*SH-coeffs/s", "value": tot_units / (tot_ms * 1e-3),
            "unit": "pole-solve*coeff/s", "n_gpus": 1, "steps": 24, "warmup": args.warmup,
            "ms_per_step": tot_ms / (24 * len(rows)), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded, SURVEY §8d)",
            "config": {"workload": "cfg3 stiffness sweep of cfg2 (T256, 36 cases x 24 steps)",
                       "trunc": 256, "grid": [cfg.nlat, cfg.nlon],
                       "l2": "flushed (256 MB write) before every timed step",
                       "cuda_graph": True},
            "all_stable": stable, "cases": rows, "clocks": clocks,
            "note": "unstable cases run all 24 steps (timed like the rest); their blow-up "
                    "step matches the oracle's (tests/golden/cfg3_verdicts.json)"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def column_breakdown(torch, eng, ccomm, flush, reps=5):
    """Rank-local device times of the column-sharded step's pieces: the
    three tendency stages (each with its slab pack/unpack copies) and one
    column-restricted pole sum; the all-to-alls are in the step time only."""
    t = eng.tend
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    acc = np.zeros(4)
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        ev[0].record()
        t.stage(0, eng.u, None, None)
        ev[1].record()
        ccomm.exchange(t, 0)
        ev[2].record()
        t.stage(1)
        ev[3].record()
        ccomm.exchange(t, 1)
        ev[4].record()
        t.stage(2, None, eng.nu[0], None)
        ev[5].record()
        torch.cuda.synchronize()
        acc[0] += ev[0].elapsed_time(ev[1])
        acc[1] += ev[2].elapsed_time(ev[3])
        acc[2] += ev[4].elapsed_time(ev[5])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.zero_()
        e0.record()
        eng.rexi.apply((2,), eng.d, eng.psi0, None, base=eng.a[None], scale=eng.dt)
        e1.record()
        e1.synchronize()
        acc[3] += e0.elapsed_time(e1)
    acc /= reps
    bd = {"synth_state": {"ms_per_launch": acc[0], "launches_per_step": 2},
          "grid_fused": {"ms_per_launch": acc[1], "launches_per_step": 2},
          "analysis": {"ms_per_launch": acc[2], "launches_per_step": 2},
          "rexi_lg": {"ms_per_launch": acc[3], "launches_per_step": 3}}
    for v in bd.values():
        v["ms_per_step"] = v["ms_per_launch"] * v["launches_per_step"]
    return bd, max(bd, key=lambda k: bd[k]["ms_per_step"])


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist

    from paper_1805_06557_b200 import _lib
    from paper_1805_06557_b200.device import ncoef, pack, to_device
    from paper_1805_06557_b200.parallel import (ColumnComm, ColumnEtdrkEngine, ColumnShard,
                                                PoleComm)
    from paper_1805_06557_b200.steppers import EtdrkStepper, RexiStepper
    from paper_1805_06557_b200.swe import LC_N, LG, L, PrognosticState, TermGroup
    from paper_1805_06557_b200.workloads import (CONFIGS, seeded_balanced_state,
                                                 seeded_linear_state)

    torch.cuda.set_device(local)
    if args.config == "cfg3":
        run_stiffness(args, rank, world)
        return
    comm = ccomm = None
    etd = CONFIGS[args.config].stepper == "lg_rexi_lc_n_etdrk"
    mode = args.shard if args.shard != "auto" else ("cols" if etd else "poles")
    if mode.startswith("cols") and not etd:
        raise SystemExit("--shard cols is the ETD2RK (cfg2) decomposition")
    # SWX_FORCE_COMM=1 routes a 1-rank run through the multi-rank path (NCCL
    # process group, pole reduce or column exchanges), to exercise it on 1 GPU
    force = os.environ.get("SWX_FORCE_COMM") == "1"
    if world > 1 or force:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if mode in ("cols-p2p", "cols-fused"):
            from paper_1805_06557_b200.parallel import SymmetricColumnComm
            ccomm = SymmetricColumnComm()
        elif mode == "cols":
            ccomm = ColumnComm()
        else:
            comm = PoleComm(deterministic=os.environ.get("SWX_FAST_REDUCE") != "1")
    lib = _lib.lib()
    w = CONFIGS[args.config]
    par = w.params
    nc = ncoef(w.trunc)
    group = TermGroup.parse(w.group)

    if ccomm is not None:
        stepper = EtdrkStepper(group, LC_N, par, w.setup)
        shard = ColumnShard(par.cfg, rank, world)
        eng = ColumnEtdrkEngine(group, LC_N, par, w.dt, stepper.coeff_set(w.dt), shard, ccomm)
        eng.use_graph = os.environ.get("SWX_COL_GRAPH") == "1"
        if mode == "cols-fused":
            ccomm.fuse(eng.tend)
        ic = seeded_balanced_state(par.cfg)
        eng.load(ic)

        def step():
            return eng.step_dev(ccomm)
        units_per_step = 3 * w.n_poles * nc
    elif etd:
        stepper = EtdrkStepper(group, LC_N, par, w.setup)
        eng = stepper.engine(w.dt, comm)
        ic = seeded_balanced_state(par.cfg)
        eng.load(ic)
        step = eng.step_dev
        units_per_step = 3 * w.n_poles * nc
    else:
        stepper = RexiStepper(group, par, w.setup)
        ic = seeded_linear_state(w.trunc, 0)
        u = to_device(pack(ic))
        out = torch.empty_like(u)
        torch.cuda.synchronize()
        t_warm = time.perf_counter()
        dr = stepper._for_dt(w.dt)[2]   # warm: guards (+ the l pivot cache), untimed
        torch.cuda.synchronize()
        t_warm = time.perf_counter() - t_warm
        if comm is not None:
            dr.set_comm(comm)

        def step_eager():
            dr.apply((0,), u[None], out[None])
            return out

        step = step_eager
        if comm is None and os.environ.get("SWX_LIN_GRAPH", "1") == "1":
            # single rank: the step's launches (pole sum, + packing and the tree
            # combine for the l chains) replayed as one CUDA graph
            gs = torch.cuda.Stream()
            gs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(gs):
                step_eager()  # warm-up: workspaces, schedules
            torch.cuda.current_stream().wait_stream(gs)
            torch.cuda.synchronize()
            lin_graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(lin_graph, stream=gs):
                step_eager()

            def step():
                lin_graph.replay()
                return out
        units_per_step = w.n_poles * nc

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    if os.environ.get("SWX_TRACE_OUT"):  # per-CTA phase marks of one step (trace build only)
        tlib = _lib.load()
        flush.zero_()
        torch.cuda.synchronize()
        tlib.swx_trace(1, None, 0)
        tlib.swx_trace_rexi(1, None, 0)
        step()
        torch.cuda.synchronize()
        tbuf = np.zeros((2, 4096, 8), dtype=np.uint64)
        tlib.swx_trace(0, tbuf[0].ctypes.data, 4096)
        tlib.swx_trace_rexi(0, tbuf[1].ctypes.data, 4096)
        np.save(os.environ["SWX_TRACE_OUT"], tbuf)
    sampler = ClockSampler(local)
    sampler.start()
    t_soak = time.perf_counter()
    while not args.profile and time.perf_counter() - t_soak < 1.0:   # steady clocks
        step()
        torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    multi = comm is not None or ccomm is not None
    if multi:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    # keep the host ahead of the GPU: a spin kernel holds the stream while the K
    # steps are enqueued behind it, so a slow host never sits between a step's
    # start event and its launches (seen: 0.206 instead of 0.166 ms/step at K = 48)
    try:
        torch.cuda._sleep(int(min(30.0, 0.4 * args.steps) * 1e-3 * 1.9e9))
    except Exception:  # private torch API: without it the loop is timed as before
        pass
    for k in range(args.steps):
        flush.zero_()                      # cold L2 for every step
        starts[k].record()
        step()
        ends[k].record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    if multi:
        dist.barrier()
    clocks = sampler.stop()
    ms_steps = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms_total = torch.tensor([sum(ms_steps)], dtype=torch.float64, device="cuda")
    if multi:
        dist.all_reduce(ms_total, op=dist.ReduceOp.MAX)
    ms_total = float(ms_total.item())
    ms_per_step = ms_total / args.steps
    value = units_per_step * args.steps / (ms_total * 1e-3)
    if args.profile:
        if rank == 0:
            print(json.dumps({"profile_mode": True, "ms_per_step": ms_per_step}), flush=True)
        return

    # ---- per-kernel breakdown (live CUDA events on the launching stream)
    from paper_1805_06557_b200.steppers import axpy

    cur = torch.cuda.current_stream()
    s_ptr = cur.cuda_stream
    breakdown = {}
    dominant = None
    if ccomm is not None:
        breakdown, dominant = column_breakdown(torch, eng, ccomm, flush)
    elif etd:
        plan = eng.plan
        reps = 5
        # with the fused grid stage, C2R+products+R2C+prep all land in "grid_fused"
        stage_names = (["synth_state", "fft_c2r", "grid_products", "grid_fused", "prep", "analysis"]
                       if plan.fused_stages() else
                       ["synth_state", "fft_c2r", "grid_products", "fft_r2c", "prep", "analysis"])
        acc = np.zeros(7)
        for _ in range(reps):
            flush.zero_()
            torch.cuda.synchronize()
            ctypes_buf = np.zeros(7, dtype=np.float64)
            _lib.check(lib.swx_sht_tendency_profile(
                plan._h, 3, eng.u.data_ptr(), eng.na.data_ptr(), plan.workspace.data_ptr(),
                plan.workspace.numel(), ctypes_buf.ctypes.data, s_ptr))
            acc += ctypes_buf
        acc /= reps
        for n, v in zip(stage_names, acc[:6]):
            if v > 0.0:  # stages the plan's path does not run report 0
                breakdown[n] = {"ms_per_launch": v, "launches_per_step": 2}
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        busy = torch.empty(1024 * 1024 * 1024, dtype=torch.uint8, device="cuda")

        def timed(fn):
            # a 1 GiB memset ahead of e0 keeps the GPU busy while Python issues
            # fn(), so the event interval is device time only (and L2 is cold)
            tt = []
            for _ in range(reps):
                busy.zero_()
                e0.record()
                fn()
                e1.record()
                e1.synchronize()
                tt.append(e0.elapsed_time(e1))
            return sum(tt) / len(tt)
        eng.pair_in[0].copy_(eng.u)
        eng.pair_in[1].copy_(eng.na)
        # rank-local pole sums (the cross-rank reduce is timed in the step)
        dr = eng.rexi

        fused = comm is None  # single rank: the ETD2RK axpys live in the sum epilogues

        def local_sum(ks, rhs, out, base=None):
            b, preps = dr.betas_for(ks)
            for prep, nd in zip(preps, dr.nodes):  # this rank's tree nodes
                dr.solver.rexi_sum_prepared_dev(dr.alphas, b, prep, rhs, out, nd,
                                                comm is None, None, base, w.dt)
        # the step runs three single-RHS prepared sums: psi0(u) (side stream,
        # concurrent with N(u)), psi1(N(u)) and psi2(N(a) - N(u)), the last two
        # with the fused update out = base + dt * sum; warm caches first
        base = eng.a[None] if fused else None
        for ks, rhs, o in (((0,), eng.pair_in[0:1], eng.pair_out[0:1]),
                           ((1,), eng.pair_in[1:2], eng.pair_out[1:2]), ((2,), eng.d, eng.r2)):
            local_sum(ks, rhs, o, base if ks != (0,) else None)
        torch.cuda.synchronize()
        breakdown["rexi_lg_psi0_overlapped"] = {"ms_per_launch": timed(
            lambda: local_sum((0,), eng.pair_in[0:1], eng.pair_out[0:1])), "launches_per_step": 1}
        breakdown["rexi_lg"] = {"ms_per_launch": timed(
            lambda: local_sum((2,), eng.d, eng.r2, base)), "launches_per_step": 2}
        if not fused:
            breakdown["axpy"] = {"ms_per_launch": timed(
                lambda: axpy(w.trunc, eng.a, w.dt, eng.r2[0], eng.na)), "launches_per_step": 3}
        for v in breakdown.values():
            v["ms_per_step"] = v["ms_per_launch"] * v["launches_per_step"]
        # dominant kernel = the kernel function with the largest device time per
        # step summed over ALL its launches, as in the ncu launch list: the lg pole
        # sum counts its three launches (psi0(u), concurrent with N(u), included)
        def fn_total(k):
            return sum(v["ms_per_step"] for n, v in breakdown.items()
                       if n == k or n == k + "_psi0_overlapped")
        dominant = max((k for k in breakdown if not k.endswith("_overlapped")), key=fn_total)
        for k in breakdown:
            if not k.endswith("_overlapped"):
                breakdown[k]["ms_per_step_all_launches"] = fn_total(k)
    elif not etd:
        # the pole sum's device time with the host ahead of the GPU (a 1 GiB
        # memset before the first event, as in the ETD2RK breakdown), so a
        # launch-bound step (cfg0) reports its kernel, not its launch latency;
        # the step line above keeps the plain per-step events
        busy = torch.empty(1024 * 1024 * 1024, dtype=torch.uint8, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tt = []
        for _ in range(5):
            busy.zero_()
            e0.record()
            step()
            e1.record()
            e1.synchronize()
            tt.append(e0.elapsed_time(e1))
        del busy
        k_ms = min(ms_per_step, sum(tt) / len(tt))
        breakdown["rexi_" + w.group] = {"ms_per_launch": k_ms, "launches_per_step": 1,
                                        "ms_per_step": k_ms,
                                        "note": "device time of the step's pole-sum launches "
                                                "with the host ahead (L2 cold)"}
        dominant = "rexi_" + w.group

    # algorithmic flops per launch (SURVEY §8d conventions)
    nlat = par.cfg.nlat
    leg = 4.0 * nlat * nc  # per complex series, no symmetry credit
    import math
    nlon_t = int(_tendency_nlon(par.cfg.trunc, par.cfg.nlon))
    # fused grid stage: 4 inverse + 5 forward complex FFTs of length nlon_t per
    # latitude pair (5 N log2 N each) + 9 flops per grid point and hemisphere
    grid_flops = (nlat // 2) * (9 * 5.0 * nlon_t * math.log2(nlon_t) + 2 * 9.0 * nlon_t)
    flops = {
        "rexi_lg_psi0_overlapped": 40.0 * w.n_poles * nc,
        "rexi_lg": 40.0 * w.n_poles * nc,
        "rexi_l": 142.0 * w.n_poles * nc,
        "synth_state": 7 * leg,
        "analysis": 7 * leg,
        "grid_fused": grid_flops,
    }
    if ccomm is not None:  # rank-local shares: own columns / own latitude pairs
        a, b = eng.shard.slots()
        fc = (b - a) / nc
        pb = eng.shard.p_bounds
        fp = (min(pb[rank + 1], nlat // 2) - min(pb[rank], nlat // 2)) / (nlat // 2)
        flops = {"rexi_lg": flops["rexi_lg"] * fc, "synth_state": flops["synth_state"] * fc,
                 "analysis": flops["analysis"] * fc, "grid_fused": grid_flops * fp}
    peak64 = fp64_peak_tflops(torch, lib, _lib)
    traffic = load_traffic()
    # every step kernel's own algorithmic rate against the FP64 peak
    for k, v in breakdown.items():
        if k in flops and v.get("ms_per_launch"):
            v["algorithmic_tflops"] = flops[k] / (v["ms_per_launch"] * 1e-3) / 1e12
            v["frac_fp64"] = v["algorithmic_tflops"] / peak64
    roofline = None
    if dominant is not None and dominant in flops:
        ms = breakdown[dominant]["ms_per_launch"]
        ach = flops[dominant] / (ms * 1e-3) / 1e12
        roofline = {"kernel": dominant, "bound": "fp64", "achieved": ach, "peak": peak64,
                    "unit": "TFLOP/s", "frac": ach / peak64,
                    "peak_source": "measured on this GPU by bench.py (swx_fp64_fma_probe, "
                                   "DFMA); MEASURED_PEAKS.json has no FP64 entry",
                    "algorithmic_flops_per_launch": flops[dominant],
                    # per-launch DRAM bytes from profiles/traffic.json: cfg2 keys are
                    # plain kernel names, other configs carry a _<config> suffix
                    "traffic": traffic.get(f"{dominant}_{args.config}",
                                           traffic.get(dominant) if args.config == "cfg2"
                                           else None)}
    elif dominant is not None:
        ms = breakdown[dominant]["ms_per_launch"]
        roofline = {"kernel": dominant, "bound": "fp64", "achieved": None, "peak": peak64,
                    "unit": "TFLOP/s", "frac": None, "ms_per_launch": ms, "traffic": None}
    # the l chains with the warm-time pivot cache stream 64 B per pole-solve x
    # coefficient (two 16 B pivots per chain position, read in both sweeps,
    # SURVEY §8d "factor-caching design"): HBM-bound; the FP64 figure moves
    # to "fp64" inside the line
    if roofline and dominant == "rexi_l" and not etd and (_l_cache_bytes(dr) or 0) > 0:
        ms = breakdown[dominant]["ms_per_launch"]
        alg_bytes = 64.0 * units_per_step / world
        hbm_peak = _hbm_peak()
        ach_gbs = alg_bytes / (ms * 1e-3) / 1e9
        fp64 = {k: roofline[k] for k in ("achieved", "peak", "unit", "frac")}
        roofline = {"kernel": dominant, "bound": "hbm", "achieved": ach_gbs, "peak": hbm_peak,
                    "unit": "GB/s", "frac": ach_gbs / hbm_peak,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)",
                    "algorithmic_bytes_per_launch": alg_bytes,
                    "traffic": traffic.get("rexi_l_" + args.config), "fp64": fp64}

    # ---- cfg4: SH transform round trip of the seeded phi' field (SURVEY §8d:
    # synthesis then analysis, 2 x (4 nlat ncoef + 2.5 nlon log2(nlon) nlat) flops)
    sh_rt = None
    if args.config == "cfg4":
        from paper_1805_06557_b200.sphere import plan_for
        plan = plan_for(par.cfg)
        phi = u[0:1].contiguous()
        grid = plan.synthesis_dev(phi)
        back = plan.analysis_dev(grid)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tt = []
        for _ in range(5):
            flush.zero_()
            e0.record()
            plan.synthesis_dev(phi, grid)
            plan.analysis_dev(grid, back)
            e1.record()
            e1.synchronize()
            tt.append(e0.elapsed_time(e1))
        import math
        nlat_, nlon_ = par.cfg.nlat, par.cfg.nlon
        fl = 2 * (4.0 * nlat_ * nc + 2.5 * nlon_ * math.log2(nlon_) * nlat_)
        ms_rt = min(tt)
        err = float((back - phi).abs().max() / phi.abs().max())
        sh_rt = {"ms": ms_rt, "coeffs_per_s": nc / (ms_rt * 1e-3),
                 "algorithmic_flops": fl, "tflops": fl / (ms_rt * 1e-3) / 1e12,
                 "rel_linf_round_trip": err, "path": "on-the-fly Legendre recurrence (no table at T1279)"}
        if multi:  # the same round trip column/latitude-sharded over the ranks
            from paper_1805_06557_b200.parallel import ShardedTransforms
            cc = ColumnComm()
            xs = ShardedTransforms(plan, ColumnShard(par.cfg, rank, world))
            tt = []
            for _ in range(5):
                flush.zero_()
                dist.barrier()
                e0.record()
                xs.synthesis(cc, phi, grid)
                xs.analysis(cc, grid, back)
                e1.record()
                e1.synchronize()
                tt.append(e0.elapsed_time(e1))
            tm = torch.tensor([min(tt)], dtype=torch.float64, device="cuda")
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            sh_rt["sharded"] = {"ms": float(tm.item()), "ranks": world,
                                "decomposition": "columns (Legendre) x latitude pairs (FFT), "
                                                 "one all-to-all per transform"}

    # ---- end to end through the public API (host numpy in, host numpy out)
    e2e = None
    if not args.no_e2e and ccomm is not None:
        # every rank: host pack + H2D of the full state, the sharded step, the
        # column all-gather and D2H + unpack of the full state
        from paper_1805_06557_b200.device import HostStage
        stage = HostStage(w.trunc)
        st_host = PrognosticState.from_stack(ic, par.cfg)
        n_e2e = max(3, min(args.steps, 20))
        tt = []
        for k in range(n_e2e + 1):
            dist.barrier()
            t0 = time.perf_counter()
            stage.upload(st_host, eng.u)
            eng.step_dev(ccomm)
            full = ccomm.gather_columns(eng.u, eng.shard)
            f = stage.download(full)
            tt.append(time.perf_counter() - t0)
            st_host = PrognosticState.from_stack(np.stack(f), par.cfg)
        sec = torch.tensor([sum(tt[1:]) / n_e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(sec, op=dist.ReduceOp.MAX)
        sec = float(sec.item())
        e2e = {"value": units_per_step / sec, "unit": "pole-solve*coeff/s",
               "ms_per_step": sec * 1e3, "h2d_bytes_per_step": 3 * nc * 16,
               "d2h_bytes_per_step": 3 * nc * 16,
               "api": "ColumnEtdrkEngine (host state in, column all-gather, host state out)"}
    if not args.no_e2e and comm is None and ccomm is None:
        st_host = PrognosticState.from_stack(ic, par.cfg)
        n_e2e = max(3, min(args.steps, 20))
        st_host = stepper.step(st_host, w.dt)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            st_host = stepper.step(st_host, w.dt)
        sec = (time.perf_counter() - t0) / n_e2e
        e2e = {"value": units_per_step / sec, "unit": "pole-solve*coeff/s",
               "ms_per_step": sec * 1e3, "h2d_bytes_per_step": 3 * nc * 16,
               "d2h_bytes_per_step": 3 * nc * 16,
               "api": ("EtdrkStepper.step(PrognosticState, dt)" if etd
                       else "RexiStepper.step(PrognosticState, dt)")}

    # ---- CPU baseline: the oracle on this host, bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not (etd and w.trunc > 341):
        from oracle import layout as olay
        from oracle import rexi as orx
        from oracle import sht as osh
        from oracle import stepping as ost

        model = orx.Model(w.trunc, w.phibar)
        if etd:
            grid = osh.grid_for(w.trunc)
            sets = {k: ost.contour_coeffs(k, w.p0, w.p1, w.n_poles) for k in (0, 1, 2)}
            t0 = time.perf_counter()
            ost.etdrk2_step(model, grid, w.dt, sets, ic)
            sec = time.perf_counter() - t0
            sample = f"1 full ETD2RK step of {w.name} (numpy/scipy oracle)"
        else:
            a, b = ost.contour_coeffs(0, w.p0, w.p1, w.n_poles)
            n_s = w.n_poles if w.trunc <= 128 else 8
            fac = orx.LFactors(model, w.dt) if w.group == "l" else None
            t0 = time.perf_counter()
            orx.rexi_sum(w.group, model, w.dt, a[:n_s], b[:n_s], ic, fac, chunk=8)
            sec = (time.perf_counter() - t0) * w.n_poles / n_s
            sample = f"{n_s} of {w.n_poles} poles of {w.name}, scaled"
        cpu = {"value": units_per_step / sec, "unit": "pole-solve*coeff/s",
               "cores": len(os.sched_getaffinity(0)), "kind": "port", "sample": sample + PORT_NOTE}

    # kernels per step: counted from the captured step graph (ETD2RK); the linear
    # configs launch one fused pole-sum kernel (lg) or kernel + tree combine (l)
    per_step_launches = (eng.kernel_launches if etd and ccomm is None else None) or \
        ((9 if comm is None else 12) if etd else (1 if w.group == "lg" else 2))
    line = {
        "metric": "REXI pole-solves*SH-coeffs/s", "value": value, "unit": "pole-solve*coeff/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded, SURVEY §8d)",
        "config": bench_config(w),
        "run_info": {"units_per_step": units_per_step,
                   "parallelism": ((f"zonal columns sharded over {world} GPU(s) ({mode})" if ccomm
                                    else f"poles sharded over {world} GPU(s)")
                                   if multi else "1 GPU"),
                   "l2": "flushed (256 MB write) before every timed step",
                   "cuda_graph": bool(not multi and (etd or os.environ.get("SWX_LIN_GRAPH", "1") == "1")),
                   **({} if etd else {"warm_s": round(t_warm, 3),
                                      "l_pivot_cache_bytes": _l_cache_bytes(dr)})},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        **({"sh_round_trip": sh_rt} if sh_rt else {}),
        "gpu_launches": per_step_launches * args.steps,
        "clocks": clocks, "kernel_breakdown_ms": breakdown,
        "wall_s_timed_region": wall,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if multi:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
