"""Multi-process runs of the product classes with their real kernels: K
processes (gloo backend, every rank on cuda:0 -- this run has one GPU; the
collectives are staged through host memory, so no kernel waits on another
rank's kernel) drive PoleComm (tree-order reduce-scatter over aligned tree
nodes), parallel_rexi_apply, the pole-sharded ETD2RK engine, and the
column-sharded ColumnEtdrkEngine / ColumnComm.  Each must equal the single
rank bit for bit (the reference's guarantee, test_parallel.py:67-78); the
column-sharded step is also checked against the CPU oracle."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

G = 9.80616


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _params(trunc):
    from paper_1805_06557_b200.sphere import SphereConfig
    from paper_1805_06557_b200.swe import ModelParams

    return ModelParams(1e4 * G, SphereConfig.for_truncation(trunc))


def _pole_worker(rank, world, port, path):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sht as osh
        from oracle import stepping as ost
        from paper_1805_06557_b200.parallel import PoleComm, distribute_terms, parallel_rexi_apply
        from paper_1805_06557_b200.rexi import RexiSetup, coeffs_for_contour, shifted_contour_from_points
        from paper_1805_06557_b200.steppers import EtdrkStepper
        from paper_1805_06557_b200.swe import LC_N, LG, L, PrognosticState

        comm = PoleComm()
        par = _params(42)
        out = {}
        st = PrognosticState.from_stack(ost.seeded_linear_state(42, 7), par.cfg)
        for group in (LG, L):
            for n in (128, 96):
                c = coeffs_for_contour("psi0", shifted_contour_from_points(10.0, 30.0, n))
                plan = distribute_terms(n, world)
                res, bd = parallel_rexi_apply(group, st, 3600.0, c, plan, par, comm=comm)
                bd.validate()
                out[f"apply_{group.token}{n}"] = res.stack()
        # pole-sharded ETD2RK engine (DeviceRexi over the rank's tree nodes)
        par63 = _params(63)
        ic = ost.seeded_balanced_state(osh.grid_for(63))
        stepper = EtdrkStepper(LG, LC_N, par63, RexiSetup(num_poles=128))
        eng = stepper.engine(1800.0, comm)
        eng.load(ic)
        for _ in range(2):
            eng.step_dev()
        out["etd63"] = eng.u.cpu().numpy()
        np.savez(f"{path}_{rank}.npz", **out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_pole_sharded_processes_bitwise(tmp_path, world):
    from oracle import sht as osh
    from oracle import stepping as ost
    from paper_1805_06557_b200.device import pack
    from paper_1805_06557_b200.rexi import RexiSetup, coeffs_for_contour, shifted_contour_from_points
    from paper_1805_06557_b200.steppers import EtdrkStepper, rexi_step
    from paper_1805_06557_b200.swe import LC_N, LG, L, PrognosticState

    path = str(tmp_path / "res")
    mp.spawn(_pole_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    par = _params(42)
    st = PrognosticState.from_stack(ost.seeded_linear_state(42, 7), par.cfg)
    par63 = _params(63)
    eng = EtdrkStepper(LG, LC_N, par63, RexiSetup(num_poles=128)).engine(1800.0)
    eng.load(ost.seeded_balanced_state(osh.grid_for(63)))
    for _ in range(2):
        eng.step_dev()
    etd = eng.u.cpu().numpy()
    for r in range(world):
        got = np.load(f"{path}_{r}.npz")
        for group in (LG, L):
            for n in (128, 96):
                c = coeffs_for_contour("psi0", shifted_contour_from_points(10.0, 30.0, n))
                serial = rexi_step(group, st, 3600.0, c, par).stack()
                assert np.array_equal(got[f"apply_{group.token}{n}"], serial), (r, group.token, n)
        assert np.array_equal(got["etd63"], etd), r


def _col_worker(rank, world, port, path):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sht as osh
        from oracle import stepping as ost
        from paper_1805_06557_b200.parallel import ColumnComm, ColumnEtdrkEngine, ColumnShard
        from paper_1805_06557_b200.rexi import RexiSetup
        from paper_1805_06557_b200.steppers import EtdrkStepper
        from paper_1805_06557_b200.swe import LC_N, LG

        comm = ColumnComm()
        par = _params(85)
        sets = EtdrkStepper(LG, LC_N, par, RexiSetup(num_poles=128)).coeff_set(1800.0)
        eng = ColumnEtdrkEngine(LG, LC_N, par, 1800.0, sets, ColumnShard(par.cfg, rank, world),
                                comm)
        eng.load(ost.seeded_balanced_state(osh.grid_for(85)))
        steps = []
        for _ in range(2):
            eng.step_dev(comm)
            steps.append(comm.gather_columns(eng.u, eng.shard).cpu().numpy())
        np.savez(f"{path}_{rank}.npz", step1=steps[0], step2=steps[1])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_column_sharded_processes_bitwise_and_oracle(tmp_path, world):
    from conftest import rel_l2
    from oracle import layout as olay
    from oracle import rexi as orx
    from oracle import sht as osh
    from oracle import stepping as ost
    from paper_1805_06557_b200.rexi import RexiSetup
    from paper_1805_06557_b200.steppers import EtdrkStepper
    from paper_1805_06557_b200.swe import LC_N, LG

    path = str(tmp_path / "res")
    mp.spawn(_col_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    par = _params(85)
    grid = osh.grid_for(85)
    ic = ost.seeded_balanced_state(grid)
    eng = EtdrkStepper(LG, LC_N, par, RexiSetup(num_poles=128)).engine(1800.0)
    eng.load(ic)
    want = []
    for _ in range(2):
        eng.step_dev()
        want.append(eng.u.cpu().numpy())
    # the oracle's ETD2RK step (steppers.py:249-269) on the same input
    sets = {k: ost.contour_coeffs(k, 10.0, 30.0, 128) for k in (0, 1, 2)}
    ref1 = olay.pack(ost.etdrk2_step(orx.Model(85, 1e4 * G), grid, 1800.0, sets, ic))
    for r in range(world):
        got = np.load(f"{path}_{r}.npz")
        assert np.array_equal(got["step1"], want[0]), r
        assert np.array_equal(got["step2"], want[1]), r
        assert rel_l2(got["step1"], ref1) <= 1e-10, r
