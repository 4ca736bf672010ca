"""World-size-2 gloo run of the pole-sharded reduce (CPU): each rank sums its
contiguous pole block (oracle partial), PoleComm all-gathers the partials and
the fixed tree over blocks reproduces the serial tree_sum bitwise."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_path):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import rexi as orx
    from oracle import stepping as ost
    from paper_1805_06557_b200.parallel import PoleComm

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = PoleComm()
        for group, n in (("lg", 128), ("l", 16)):
            a, b = ost.contour_coeffs(0, 10.0, 30.0, n)
            st = ost.seeded_linear_state(21, seed=4)
            model = orx.Model(21, 1e4 * 9.80616)
            lo, hi = comm.pole_range(n)
            assert (lo, hi) == ((0, n // 2) if rank == 0 else (n // 2, n))
            part = orx.rexi_partial(group, model, 480.0, a, b, st, lo, hi)
            t = torch.from_numpy(np.ascontiguousarray(part))
            parts = comm.gather_parts(t).numpy()
            combined, _ = orx.realify(orx.tree_sum(parts))
            serial = orx.rexi_sum(group, model, 480.0, a, b, st, chunk=n // 2)
            if rank == 0:
                np.save(result_path + f"_{group}.npy", np.stack([combined, serial]))
    finally:
        dist.destroy_process_group()


def test_two_rank_tree_reduce_bitwise(tmp_path):
    port = _free_port()
    path = str(tmp_path / "res")
    mp.spawn(_worker, args=(2, port, path), nprocs=2, join=True)
    for group in ("lg", "l"):
        combined, serial = np.load(path + f"_{group}.npy")
        assert np.array_equal(combined, serial), group
