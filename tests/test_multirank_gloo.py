"""Multi-rank gloo runs on CPU (world size 2 and 3).

Pole shards: each rank sums its aligned tree nodes (oracle partials), the
real PoleComm exchange (all-to-all of 1/K slices, all-gather of the combined
slices) moves them, and the tree over nodes -- here the oracle's tree_sum
standing in for swx_tree_combine_flat -- reproduces the serial tree_sum
bitwise, for power-of-two and other pole / rank counts."""

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
    from paper_1805_06557_b200.parallel import PoleComm, pole_nodes

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = PoleComm()
        for group, n in (("lg", 128), ("l", 16), ("lg", 96), ("l", 12)):
            a, b = ost.contour_coeffs(0, 10.0, 30.0, n)
            st = ost.seeded_linear_state(21, seed=4)
            model = orx.Model(21, 1e4 * 9.80616)
            nodes = comm.nodes(n)
            assert nodes == pole_nodes(n, world)[1][rank]
            if world == 2 and n in (128, 16):  # power of two: the reference's blocks
                assert nodes == (((0, n // 2),) if rank == 0 else ((n // 2, n),))
            parts = np.stack([orx.rexi_partial(group, model, 480.0, a, b, st, lo, hi)
                              for lo, hi in nodes])
            recv = comm.scatter_slices(torch.from_numpy(parts), n).numpy()
            mine = torch.from_numpy(np.ascontiguousarray(orx.tree_sum(recv)))
            out = torch.empty(parts[0].shape, dtype=torch.complex128)
            comm.gather_slices(mine, out)
            combined, _ = orx.realify(out.numpy())
            if group == "l":  # one-shot tree over all n poles (the reference's order)
                sols = np.stack([orx.LFactors(model, 480.0).solve(x, st) for x in a])
                serial, _ = orx.realify(orx.tree_sum(b[:, None, None, None] * sols))
            else:
                serial = orx.rexi_sum(group, model, 480.0, a, b, st)
            if rank == 0:
                np.save(result_path + f"_{group}{n}.npy", np.stack([combined, serial]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_pole_tree_reduce_scatter_bitwise(tmp_path, world):
    port = _free_port()
    path = str(tmp_path / "res")
    mp.spawn(_worker, args=(world, port, path), nprocs=world, join=True)
    for tag in ("lg128", "l16", "lg96", "l12"):
        combined, serial = np.load(path + f"_{tag}.npy")
        assert np.array_equal(combined, serial), tag


def test_pole_nodes_partition():
    """Aligned nodes cover the poles in order; power-of-two N and K give the
    reference's distribute_terms blocks; loads balanced within 12.5 %."""
    from paper_1805_06557_b200.parallel import distribute_terms, pole_nodes

    for n in (12, 16, 96, 100, 128, 256, 1000, 1024, 2048):
        for k in range(1, 9):
            if k > n:
                continue
            size, ranges = pole_nodes(n, k)
            flat = [r for rr in ranges for r in rr]
            assert flat[0][0] == 0 and flat[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(flat, flat[1:]))
            assert all(lo % size == 0 and (hi - lo == size or hi == n) for lo, hi in flat)
            assert all(len(r) >= 1 for r in ranges)
            if n & (n - 1) == 0 and k & (k - 1) == 0:
                blocks = distribute_terms(n, k).assignments
                assert [((b[0], b[-1] + 1),) for b in blocks] == list(ranges)
            if size > 1:
                assert max(sum(h - l for l, h in r) for r in ranges) <= 1.125 * n / k


# ------------------------------------------------------------------ column shards
# The exchange protocol of the column-sharded tendency on
# real ranks: the device stages are replaced by numpy restatements of the
# same three stages (Legendre synthesis of the own columns -> latitude rows
# of every peer; grid products of the own latitude pairs -> columns of every
# peer; Legendre analysis of the own columns), moved by ColumnComm.all_to_all
# over gloo with the ColumnShard bounds of the library, then assembled by
# ColumnComm.gather_columns.  The result must equal the oracle's unsharded
# tendency_n.

def _pair_rows(nlat, a, b):
    """Latitude rows of pairs [a, b): south rows a..b-1, north rows nlat-b..nlat-a-1."""
    nh = (nlat + 1) // 2
    a, b = min(a, nh), min(b, nh)
    return np.unique(np.r_[np.arange(a, b), np.arange(nlat - b, nlat - a)]).astype(int)


def _col_worker(rank, world, port, result_path):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import layout as olay
    from oracle import sht as osh
    from oracle import stepping as ost
    from paper_1805_06557_b200.parallel import ColumnComm, ColumnShard
    from paper_1805_06557_b200.sphere import SphereConfig

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        trunc = 21
        g = osh.grid_for(trunc)
        cfg = SphereConfig.for_truncation(trunc)
        assert (cfg.nlat, cfg.nlon) == (g.nlat, g.nlon)
        shard = ColumnShard(cfg, rank, world)
        comm = ColumnComm()
        mb, pb = shard.m_bounds, shard.p_bounds
        st = ost.seeded_balanced_state(g)
        st[2] = ost.seeded_linear_state(trunc, 9)[2] * 1e-1
        T1, nlat, a_r = trunc + 1, g.nlat, g.radius
        im = 1j * g.ms[None, :]
        sec = 1.0 / g.cosl[:, None]
        rows = [_pair_rows(nlat, pb[r], pb[r + 1]) for r in range(world)]
        cols = [np.arange(mb[r], mb[r + 1]) for r in range(world)]

        def exchange(blocks):  # blocks[peer] -> numpy array for that peer
            send = [np.ascontiguousarray(blocks[s]).view(np.uint8).ravel()
                    if s != rank else np.zeros(0, np.uint8) for s in range(world)]
            sc = [x.size for x in send]
            rc = torch.tensor(sc)
            allc = [torch.zeros_like(rc) for _ in range(world)]
            dist.all_gather(allc, rc)
            rcv = [int(allc[r][rank]) for r in range(world)]
            sbuf = torch.from_numpy(np.concatenate(send) if sum(sc) else np.zeros(1, np.uint8))
            rbuf = torch.zeros(max(sum(rcv), 1), dtype=torch.uint8)
            comm.all_to_all(sbuf, sc, rbuf, rcv)
            out, o = {}, 0
            for r in range(world):
                out[r] = rbuf[o:o + rcv[r]].numpy()
                o += rcv[r]
            return out

        # stage 0: own columns, all latitudes (u, v, vort, phi' Fourier rows)
        own = np.zeros(T1)
        own[cols[rank]] = 1.0
        vort, div, phi = st[1] * own, st[2] * own, st[0] * own
        psi, chi = g.inv_laplacian(vort), g.inv_laplacian(div)
        ls = g.legendre_synthesis
        F = np.stack([(ls(chi * im, "p") * sec - ls(psi, "h")) / a_r,
                      (ls(psi * im, "p") * sec + ls(chi, "h")) / a_r,
                      ls(vort, "p"), ls(phi, "p")])
        got = exchange({s: F[:, rows[s]][:, :, cols[rank]] for s in range(world)})
        Fr = np.zeros((4, rows[rank].size, T1), complex)
        for r in range(world):
            blk = F[:, rows[rank]][:, :, cols[r]] if r == rank else \
                got[r].view(complex).reshape(4, rows[rank].size, cols[r].size)
            Fr[:, :, cols[r]] = blk
        # stage 1: own latitude rows -> grids -> products -> Fourier rows
        half = np.zeros((4, rows[rank].size, g.nlon // 2 + 1), complex)
        half[..., :T1] = Fr
        u, v, z, p = np.fft.irfft(half, n=g.nlon, axis=2) * g.nlon
        prods = np.stack([p * u, p * v, z * u, z * v, 0.5 * (u * u + v * v)])
        Gr = np.fft.fft(prods, axis=2)[..., :T1] * g.dlon
        got = exchange({r: Gr[:, :, cols[r]] for r in range(world)})
        Gc = np.zeros((5, nlat, T1), complex)
        for s in range(world):
            blk = Gr[:, :, cols[rank]] if s == rank else \
                got[s].view(complex).reshape(5, rows[s].size, cols[rank].size)
            Gc[:, rows[s][:, None], cols[rank][None, :]] = blk
        # stage 2: own columns, Legendre analysis (vortdiv_from_uv, sphere.py:405-430)
        la = g.legendre_analysis
        woc = g.w / g.cosl

        def vortdiv(fu, fv):
            return ((im * la(fv, "p", woc) + la(fu, "h", g.w)) / a_r,
                    (im * la(fu, "p", woc) - la(fv, "h", g.w)) / a_r)

        _, div_pf = vortdiv(Gc[0], Gc[1])
        curl_zf, div_zf = vortdiv(Gc[2], Gc[3])
        ke = la(Gc[4], "p", g.w)
        res = np.stack([-div_pf, -div_zf, curl_zf - g.laplacian(ke)]) * own
        full = comm.gather_columns(torch.from_numpy(olay.pack(res)), shard).numpy()
        if rank == 0:
            np.save(result_path, np.stack([full, olay.pack(g.tendency_n(st))]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_column_sharded_tendency_exchange(tmp_path, world):
    port = _free_port()
    path = str(tmp_path / "col.npy")
    mp.spawn(_col_worker, args=(world, port, path), nprocs=world, join=True)
    got, ref = np.load(path)
    err = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
    assert err <= 1e-12, err
