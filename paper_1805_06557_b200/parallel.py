"""Pole-parallel REXI over ranks (one process per GPU) with a deterministic
reduce (host mirror of swerexi.parallel).

API-compatible with /root/reference/pkg/src/swerexi/parallel.py:
``WorkPlan`` (30-44), ``distribute_terms`` (47-58), ``TimingBreakdown``
(61-97), ``parallel_rexi_apply`` (100-182), ``amdahl_report`` (185-214).

The reference's "workers" are threads of one process with a timed no-op
broadcast and an in-process ``tree_sum`` reduce.  Here a worker is a rank
(one per GPU, ``torch.distributed`` over NCCL): every rank already holds the
input state (no broadcast), sums its contiguous pole block on its GPU, and
the blocks are reduced either
  * deterministically: all-gather of the K block partials, then the fixed
    tree over blocks on the device (``swx_tree_combine``).  For power-of-two
    N and K the blocks are aligned subtrees of tree_sum, so the result is
    bitwise identical for every K (test_parallel.py:67-78), or
  * fast: one NCCL all-reduce (within ~1e-13 of the tree; the reference's
    ``deterministic=False``).
then realified.  Within one process (K = 1 rank) ``workers`` only selects
the reference's timing schema: the fused kernel already covers all poles.
"""

from __future__ import annotations

import dataclasses
import json
import time

import numpy as np

from . import _lib
from .device import ncoef, pack, ptr, stream_ptr, to_device, unpack
from .errors import ConfigurationError, SolverError
from .rexi import RexiCoefficients
from .solvers import ShiftedLinearSolver, get_solver
from .swe import ModelParams, PrognosticState, TermGroup

BREAKDOWN_SLACK = 0.05


@dataclasses.dataclass(frozen=True)
class WorkPlan:
    assignments: tuple[tuple[int, ...], ...]
    num_workers: int
    num_terms: int

    def __post_init__(self):
        flat = [i for chunk in self.assignments for i in chunk]
        if sorted(flat) != list(range(self.num_terms)):
            raise ConfigurationError("assignments must partition the term indices")
        sizes = [len(c) for c in self.assignments]
        if sizes and max(sizes) - min(sizes) > 1:
            raise ConfigurationError("work plan is unbalanced")


def distribute_terms(num_terms: int, num_workers: int) -> WorkPlan:
    """Contiguous partition, sizes differing by at most one (front-loaded)."""
    if num_terms < 1 or num_workers < 1:
        raise ConfigurationError("need at least one term and one worker")
    base, extra = divmod(num_terms, num_workers)
    bounds = np.concatenate([[0], np.cumsum([base + (w < extra) for w in range(num_workers)])])
    return WorkPlan(tuple(tuple(range(bounds[w], bounds[w + 1])) for w in range(num_workers)),
                    num_workers, num_terms)


@dataclasses.dataclass
class TimingBreakdown:
    overall: float
    nonlinearities: float
    rexi_total: float
    broadcast: float
    term_solves: float
    reduce: float

    def validate(self):
        for name, value in dataclasses.asdict(self).items():
            if value < 0:
                raise ConfigurationError(f"negative timing for {name}")
        if self.broadcast + self.term_solves + self.reduce > self.rexi_total * (1 + BREAKDOWN_SLACK):
            raise ConfigurationError("REXI sub-categories exceed the REXI total")
        if self.rexi_total > self.overall * (1 + BREAKDOWN_SLACK):
            raise ConfigurationError("REXI total exceeds the overall time")
        return self

    def merged_with(self, other: "TimingBreakdown") -> "TimingBreakdown":
        return TimingBreakdown(*(getattr(self, f.name) + getattr(other, f.name)
                                 for f in dataclasses.fields(self)))

    def to_json(self, num_workers: int, num_terms: int, ensemble_index: int) -> str:
        d = dataclasses.asdict(self)
        d.update({"K": num_workers, "N": num_terms, "ensemble_index": ensemble_index})
        return json.dumps(d, sort_keys=True)


def pole_nodes(n_poles: int, world: int) -> tuple[int, tuple]:
    """Aligned subtrees of ``tree_sum`` (steppers.py:157-172) dealt to ranks.

    Level h of the reference's pairwise tree (odd tails carried) holds the
    tree sums of the aligned pole blocks [j 2^h, (j+1) 2^h) clipped to N,
    and the rest of the reduction is ``tree_sum`` over those nodes.  Ranks
    get contiguous runs of nodes (``distribute_terms`` over the node count)
    at the coarsest level whose pole counts are balanced within 12.5 %; a
    rank sums each of its nodes separately, so the combine over all nodes
    reproduces the serial tree bit for bit for EVERY N and K.  For
    power-of-two N and K this is one node per rank, the reference's own
    contiguous blocks (parallel.py:47-58).  Returns (node size, per-rank
    tuples of (lo, hi) pole ranges).
    """
    if n_poles < 1 or world < 1:
        raise ConfigurationError("need at least one pole and one rank")
    if world > n_poles:
        raise ConfigurationError("more ranks than REXI poles")
    h = max((n_poles // world).bit_length() - 1, 0)
    while True:
        size = 1 << h
        n_nodes = -(-n_poles // size)
        assign = distribute_terms(n_nodes, world).assignments
        ranges = tuple(tuple((j * size, min((j + 1) * size, n_poles)) for j in a) for a in assign)
        load = max(sum(b - a for a, b in r) for r in ranges)
        if h == 0 or load <= 1.125 * n_poles / world:
            return size, ranges
        h -= 1


class _Collectives:
    """torch.distributed calls on device tensors.  NCCL takes them as they
    are; with the gloo backend (CPU collectives: the multi-process tests
    that run every rank on one GPU) the tensors are staged through host
    memory -- the device kernels around the exchange are the same."""

    def _init_group(self, group):
        import torch.distributed as dist

        if not dist.is_initialized():
            raise ConfigurationError(
                f"{type(self).__name__} needs an initialised torch.distributed group")
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.staged = dist.get_backend(group) == "gloo"

    def _a2a(self, out, inp, out_splits, in_splits):
        """all_to_all_single on flat tensors (element splits)."""
        if self.staged and inp.is_cuda:
            o = out.new_empty(out.shape, device="cpu")
            self.dist.all_to_all_single(o, inp.cpu(), list(out_splits), list(in_splits),
                                        group=self.group)
            out.copy_(o)
        else:
            self.dist.all_to_all_single(out, inp, list(out_splits), list(in_splits),
                                        group=self.group)

    def _ag(self, out, inp):
        """all_gather_into_tensor on flat tensors."""
        if self.staged and inp.is_cuda:
            o = out.new_empty(out.shape, device="cpu")
            self.dist.all_gather_into_tensor(o, inp.cpu(), group=self.group)
            out.copy_(o)
        else:
            self.dist.all_gather_into_tensor(out, inp, group=self.group)

    def _ar(self, t):
        if self.staged and t.is_cuda:
            c = t.cpu()
            self.dist.all_reduce(c, group=self.group)
            t.copy_(c)
        else:
            self.dist.all_reduce(t, group=self.group)


def torch_view_real(t):
    """Flat float64 view of a complex128 tensor (collectives move reals)."""
    import torch

    return torch.view_as_real(t).reshape(-1) if t.is_complex() else t.reshape(-1)


class PoleComm(_Collectives):
    """Rank-level pole sharding over an initialised torch.distributed group.

    Each rank sums its aligned tree nodes (``pole_nodes``) un-realified; the
    deterministic reduce is a tree-order reduce-scatter: one all-to-all
    hands rank s the s-th 1/K slice of every node partial, rank s combines
    its slice over all nodes in tree order on the device
    (``swx_tree_combine_flat``), one all-gather assembles the slices, and
    the m = 0 column is realified.  Each rank moves 2 (K-1)/K of a state
    (per node it owns) instead of the K-1 states of an all-gather of the
    partials, and the result is bitwise the serial ``tree_sum`` for every
    K.  ``deterministic=False`` is the reference's fast path: the
    ``distribute_terms`` blocks and one all-reduce (~1e-13 of the tree).
    """

    def __init__(self, group=None, deterministic: bool = True):
        self._init_group(group)
        self.deterministic = deterministic

    def nodes(self, n_poles: int, deterministic: bool | None = None) -> tuple:
        """This rank's pole ranges: aligned tree nodes (deterministic) or its
        distribute_terms block."""
        det = self.deterministic if deterministic is None else deterministic
        if not det:
            chunk = distribute_terms(n_poles, self.world).assignments[self.rank]
            if not chunk:
                raise ConfigurationError("more ranks than REXI poles")
            return ((chunk[0], chunk[-1] + 1),)
        return pole_nodes(n_poles, self.world)[1][self.rank]

    def pole_range(self, n_poles: int, deterministic: bool | None = None) -> tuple[int, int]:
        """Contiguous pole span of this rank (the union of its nodes)."""
        nd = self.nodes(n_poles, deterministic)
        return nd[0][0], nd[-1][1]

    # -- the exchange (device-agnostic: tensors of any device) ---------------
    def scatter_slices(self, parts, n_poles: int):
        """Reduce-scatter exchange: ``parts`` (M_r, ...) complex node partials
        of this rank -> (M, S) complex: the rank's slice (S values) of every
        node partial of every rank, in node (= tree) order."""
        import torch

        counts = [len(r) for r in pole_nodes(n_poles, self.world)[1]]
        m_r = parts.shape[0]
        if m_r != counts[self.rank]:
            raise ConfigurationError("node partials do not match the pole partition")
        E = parts[0].numel()
        K = self.world
        S = -(-E // K)
        flat = parts.reshape(m_r, E)
        if E != K * S:
            pad = torch.zeros((m_r, K * S), dtype=parts.dtype, device=parts.device)
            pad[:, :E] = flat
            flat = pad
        send = flat.view(m_r, K, S).transpose(0, 1).contiguous()  # (K dest, M_r, S)
        recv = torch.empty((sum(counts), S), dtype=parts.dtype, device=parts.device)
        self._a2a(torch_view_real(recv), torch_view_real(send),
                  [2 * c * S for c in counts], [2 * m_r * S] * K)
        return recv

    def gather_slices(self, mine, out):
        """All-gather of the combined slices into ``out`` (E complex values)."""
        import torch

        E = out.numel()
        S = mine.numel()
        full = torch.empty(self.world * S, dtype=mine.dtype, device=mine.device)
        self._ag(torch_view_real(full), torch_view_real(mine))
        out.view(-1).copy_(full[:E])
        return out

    # -- device reduce ---------------------------------------------------------
    def reduce_nodes_realify(self, parts, out, trunc: int, n_poles: int, stream=None,
                             deterministic: bool | None = None):
        """out <- realify(tree-order reduce over ranks of the node partials
        ``parts`` (M_r, n_states, 3, ncoef)); ``out`` may alias parts[0]."""
        import torch

        det = self.deterministic if deterministic is None else deterministic
        n_states = out.numel() // (3 * ncoef(trunc))
        lib = _lib.load()
        with torch.cuda.stream(stream) if stream is not None else _null():
            if det:
                recv = self.scatter_slices(parts, n_poles)
                mine = torch.empty(recv.shape[1], dtype=recv.dtype, device=recv.device)
                _lib.check(lib.swx_tree_combine_flat(recv.shape[1], recv.shape[0], ptr(recv),
                                                     ptr(mine), stream_ptr(stream)))
                self.gather_slices(mine, out)
            else:
                if parts.shape[0] != 1:
                    raise ConfigurationError("the fast reduce takes one block per rank")
                if out.data_ptr() != parts.data_ptr():
                    out.copy_(parts[0])
                self._ar(torch_view_real(out))
            _lib.check(lib.swx_tree_combine(trunc, n_states, 1, ptr(out), 1, ptr(out),
                                            stream_ptr(stream)))
        return out

    def reduce_realify(self, partial, trunc: int, n_poles: int, stream=None,
                       deterministic: bool | None = None):
        """In-place: partial <- realify(reduce over ranks of partial), one
        node per rank."""
        return self.reduce_nodes_realify(partial[None], partial, trunc, n_poles, stream,
                                         deterministic)


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def parallel_rexi_apply(group: TermGroup, state, dt: float, coeffs: RexiCoefficients,
                        plan: WorkPlan, params: ModelParams,
                        solver: ShiftedLinearSolver | None = None,
                        deterministic: bool = True, comm: PoleComm | None = None):
    """REXI sum with the reference's timing schema (parallel.py:100-182).

    Single rank: deterministic=True is one fused pass over all poles
    (bitwise equal to ``rexi_step`` for every ``plan``); deterministic=False
    sums the plan's chunks separately and accumulates them in chunk order,
    like the reference's fast path.  With ``comm`` the poles are sharded over
    ranks instead (see module docstring).
    """
    import torch

    if plan.num_terms != coeffs.num_terms:
        raise ConfigurationError("work plan does not match the coefficient count")
    t_start = time.perf_counter()
    if solver is None:
        solver = get_solver(group.token, dt, params)
    try:
        solver.warm(coeffs.alphas)
    except SolverError as exc:
        raise SolverError(f"terms {tuple(range(coeffs.num_terms))}: {exc}") from exc
    cfg = params.cfg
    t0 = time.perf_counter()
    stack = np.stack([state.phi_pert.coeffs, state.vort.coeffs, state.div.coeffs]).astype(
        np.complex128)
    rhs = to_device(pack(stack))[None]
    betas = to_device(np.asarray(coeffs.betas).reshape(1, -1))
    torch.cuda.synchronize()
    t_broadcast = time.perf_counter() - t0

    t0 = time.perf_counter()
    if comm is not None:
        nodes = comm.nodes(coeffs.num_terms, deterministic)
        parts = torch.empty((len(nodes),) + tuple(rhs.shape), dtype=rhs.dtype, device=rhs.device)
        for j, (lo, hi) in enumerate(nodes):
            solver.rexi_sum_dev(coeffs.alphas, betas, rhs, parts[j], pole_range=(lo, hi),
                                realify=False)
        torch.cuda.synchronize()
        t_solves = time.perf_counter() - t0
        t0 = time.perf_counter()
        out = parts[0]
        comm.reduce_nodes_realify(parts, out, cfg.trunc, coeffs.num_terms,
                                  deterministic=deterministic)
    elif deterministic:
        out = solver.rexi_sum_dev(coeffs.alphas, betas, rhs, realify=True)
        torch.cuda.synchronize()
        t_solves = time.perf_counter() - t0
        t0 = time.perf_counter()
    else:
        parts = [solver.rexi_sum_dev(coeffs.alphas, betas, rhs, pole_range=(c[0], c[-1] + 1),
                                     realify=False)
                 for c in plan.assignments if c]
        torch.cuda.synchronize()
        t_solves = time.perf_counter() - t0
        t0 = time.perf_counter()
        out = parts[0]
        for p in parts[1:]:
            out = out + p
        _lib.check(_lib.load().swx_tree_combine(cfg.trunc, 1, 1, ptr(out), 1, ptr(out),
                                                stream_ptr()))
    result = PrognosticState.from_stack(unpack(out[0].cpu().numpy(), cfg.trunc), cfg)
    t_reduce = time.perf_counter() - t0
    t_end = time.perf_counter()
    bd = TimingBreakdown(overall=t_end - t_start, nonlinearities=0.0,
                         rexi_total=t_end - t_start, broadcast=t_broadcast,
                         term_solves=t_solves, reduce=t_reduce).validate()
    return result, bd


def amdahl_report(breakdowns: dict) -> list[dict]:
    if 1 not in breakdowns:
        raise ConfigurationError("amdahl_report needs a K=1 baseline breakdown")
    if len(breakdowns) < 2:
        raise ConfigurationError("need breakdowns for at least two worker counts")
    base = breakdowns[1]
    par = base.term_solves / base.overall if base.overall > 0 else 0.0
    ser = 1.0 - par
    rows = []
    for k in sorted(breakdowns):
        b = breakdowns[k]
        rows.append({
            "K": k,
            "overall": b.overall,
            "projected_speedup": 1.0 / (ser + par / k),
            "measured_speedup": base.overall / b.overall if b.overall > 0 else float("nan"),
            "serial_fraction": ser,
            "max_speedup": 1.0 / ser if ser > 0 else float("inf"),
        })
    return rows


# ----------------------------------------------------------------------
# Column-sharded N term and ETD2RK over ranks
#
# The reference replicates the non-linear tendency on every worker
# (parallel.py:185-214: the Amdahl serial part).  Here rank r owns the zonal
# columns [m_bounds[r], m_bounds[r+1]) of the packed state (a contiguous slot
# range: the layout is m-major) and the latitude pairs [p_bounds[r],
# p_bounds[r+1]).  A tendency is three device stages with two all-to-all
# exchanges in between (swx_sht_tendency_shard); the lg pole sums are
# diagonal in (l, m), so they run on the own columns with no exchange at all.
# An ETD2RK step therefore needs four all-to-alls and no all-reduce, and the
# state stays column-sharded between steps.

def shard_bounds(trunc: int, nlat: int, nranks: int) -> tuple[tuple, tuple]:
    """Host mirror of swx_shard_init: columns balanced by length T+1-m,
    latitude pairs split evenly, padding pairs (up to a multiple of 16) on
    the last rank."""
    if nranks < 1 or nranks > _lib.SWX_MAX_RANKS:
        raise ConfigurationError("bad number of ranks")
    total = (trunc + 1) * (trunc + 2) // 2
    mb, acc, m = [0], 0, 0
    for r in range(1, nranks):
        target = (total * r + nranks // 2) // nranks
        while m <= trunc and acc + (trunc + 1 - m) // 2 < target:
            acc += trunc + 1 - m
            m += 1
        mb.append(m)
    mb.append(trunc + 1)
    nh = (nlat + 1) // 2
    nt16 = (nh + 15) // 16 * 16
    pb = [nh * r // nranks for r in range(nranks)] + [nt16]
    return tuple(mb), tuple(pb)


def column_slots(trunc: int, m0: int, m1: int) -> tuple[int, int]:
    """Packed slot range [s0, s1) of columns [m0, m1) (slot(l, m) m-major)."""
    off = lambda m: m * (trunc + 1) - m * (m - 1) // 2  # noqa: E731
    return off(m0), off(m1)


class ColumnShard:
    """One rank's share of a column-sharded plan (the swx_shard struct)."""

    def __init__(self, cfg, rank: int, nranks: int):
        import ctypes

        self.cfg = cfg
        self.rank, self.nranks = int(rank), int(nranks)
        self.c = _lib.Shard()
        _lib.check(_lib.load().swx_shard_init(ctypes.byref(self.c), cfg.trunc, cfg.nlat,
                                              self.nranks, self.rank))
        self.m_bounds = tuple(self.c.m_bounds[: self.nranks + 1])
        self.p_bounds = tuple(self.c.p_bounds[: self.nranks + 1])

    @property
    def columns(self) -> tuple[int, int]:
        return self.m_bounds[self.rank], self.m_bounds[self.rank + 1]

    def slots(self, rank: int | None = None) -> tuple[int, int]:
        r = self.rank if rank is None else rank
        return column_slots(self.cfg.trunc, self.m_bounds[r], self.m_bounds[r + 1])


class ColumnComm(_Collectives):
    """torch.distributed plumbing of the column shards (NCCL on GPUs)."""

    def __init__(self, group=None):
        self._init_group(group)

    def workspace(self, nbytes: int, device):
        """The workspace a ShardedTendency of this communicator uses (None: its own)."""
        return None

    def exchange(self, tend, ex: int, stream=None):
        """Exchange ``ex`` of a sharded stage pipeline (NCCL all-to-all of the slabs)."""
        self.all_to_all(*tend.slabs(ex))

    def all_to_all(self, send, send_counts, recv, recv_counts):
        """Byte slabs ordered by peer (swx_sht_shard_counts order)."""
        if self.world == 1:  # the self slab never travels
            return
        self._a2a(recv[: sum(recv_counts)], send[: sum(send_counts)], recv_counts, send_counts)

    def gather_columns(self, state, shard: ColumnShard):
        """Full packed state(s) on every rank from the ranks' own columns.
        ``state``: (..., 3, ncoef); returns a new tensor of the same shape."""
        import torch

        lead = state.shape[:-1]
        spans = [shard.slots(r) for r in range(self.world)]
        width = max(b - a for a, b in spans)
        a, b = spans[self.rank]
        mine = torch.zeros(lead + (width,), dtype=state.dtype, device=state.device)
        mine[..., : b - a] = state[..., a:b]
        flat = torch.view_as_real(mine).reshape(-1) if mine.is_complex() else mine.reshape(-1)
        allp = torch.empty((self.world * flat.numel(),), dtype=flat.dtype, device=state.device)
        self._ag(allp, flat)
        if mine.is_complex():
            allp = torch.view_as_complex(allp.view(-1, 2))
        allp = allp.view((self.world,) + tuple(mine.shape))
        out = torch.empty_like(state)
        for r, (a, b) in enumerate(spans):
            out[..., a:b] = allp[r][..., : b - a]
        return out


class ShardedTendency:
    """tendency_group of one rank's columns (swx_sht_tendency_shard).

    Owns its workspace and exchange slabs.  ``stage(k, ...)`` runs device
    stage k; ``slabs(ex)`` gives (send, send_counts, recv, recv_counts) of
    exchange ``ex`` for the caller's all-to-all.
    """

    def __init__(self, plan, shard: ColumnShard, atoms: int, workspace=None):
        import ctypes

        import torch

        self.plan, self.shard, self.atoms = plan, shard, int(atoms)
        lib = self._lib = _lib.lib()
        dev = plan.device
        # ``workspace``: caller-provided (e.g. symmetric memory for direct pushes)
        self.workspace = (torch.empty(plan.workspace.numel(), dtype=torch.uint8, device=dev)
                          if workspace is None else workspace)
        self.direct = False  # True: stages leave the exchanges to push()
        self.pmap = None     # device peer map: stages store into the owners' workspaces
        K = shard.nranks
        self.counts = []
        size = 1
        for ex in (0, 1):
            snd, rcv = (ctypes.c_size_t * K)(), (ctypes.c_size_t * K)()
            n = lib.swx_sht_shard_counts(plan._h, ctypes.byref(shard.c), ex, self.atoms, snd, rcv)
            if n == 0:
                _lib.check(_lib.SWX_ERR_CONFIG)
            self.counts.append((tuple(snd), tuple(rcv)))
            size = max(size, int(n))
        self.send = torch.empty(size, dtype=torch.uint8, device=dev)
        self.recv = torch.empty(size, dtype=torch.uint8, device=dev)

    def slabs(self, ex: int):
        s, r = self.counts[ex]
        return self.send, s, self.recv, r

    def stage(self, k: int, state=None, out=None, sub=None, stream=None):
        import ctypes

        if self.pmap is not None:  # fused: peer stores from the stage epilogues
            _lib.check(self._lib.swx_sht_tendency_shard_peer(
                self.plan._h, int(k), self.atoms, ctypes.byref(self.shard.c), self.pmap,
                ptr(state) if state is not None else 0, ptr(sub) if sub is not None else 0,
                ptr(out) if out is not None else 0, ptr(self.workspace),
                self.workspace.numel(), stream_ptr(stream)))
            return
        slabs = (0, 0) if self.direct else (ptr(self.recv), ptr(self.send))
        _lib.check(self._lib.swx_sht_tendency_shard(
            self.plan._h, int(k), self.atoms, ctypes.byref(self.shard.c),
            ptr(state) if state is not None else 0, ptr(sub) if sub is not None else 0,
            ptr(out) if out is not None else 0, *slabs,
            ptr(self.workspace), self.workspace.numel(), stream_ptr(stream)))

    def use_peer_stores(self, peer_ws):
        """Fuse the exchanges into the stage epilogues: the kernels store into
        the owners' workspaces (``peer_ws``: device addresses of every rank's
        workspace, this rank's included)."""
        import ctypes

        addrs = (ctypes.c_uint64 * self.shard.nranks)(*[int(a) for a in peer_ws])
        h = ctypes.c_void_p()
        _lib.check(self._lib.swx_sht_peer_map_create(self.plan._h, ctypes.byref(self.shard.c),
                                                     addrs, ctypes.byref(h)))
        self.pmap = h

    def __del__(self):
        if getattr(self, "pmap", None) is not None:
            try:
                self._lib.swx_sht_peer_map_destroy(self.pmap)
            except Exception:
                pass

    def push(self, ex: int, peer_ws, stream=None):
        """Direct exchange: this rank's blocks of ``ex`` into every peer's
        workspace (``peer_ws``: device addresses of the ranks' workspaces)."""
        import ctypes

        addrs = (ctypes.c_uint64 * self.shard.nranks)(*[int(a) for a in peer_ws])
        _lib.check(self._lib.swx_sht_shard_push(
            self.plan._h, ctypes.byref(self.shard.c), int(ex), self.atoms, ptr(self.workspace),
            addrs, stream_ptr(stream)))

    def phases(self, state, out, sub=None, stream=None):
        """Generator: runs the stages, yielding (self, ex) where exchange
        ``ex`` must happen before the next stage."""
        self.stage(0, state, None, None, stream)
        yield self, 0
        self.stage(1, None, None, None, stream)
        yield self, 1
        self.stage(2, None, out, sub, stream)

    def run(self, comm: ColumnComm, state, out, sub=None, stream=None):
        for t, ex in self.phases(state, out, sub, stream):
            comm.exchange(t, ex, stream)
        return out


def virtual_exchange(ranks, ex: int):
    """All-to-all between co-resident shards of ONE device (tests and the
    single-GPU check of the multi-rank path): rank r's slab for peer s is
    copied into peer s's receive slab at r's position.  Stream-ordered on
    the current stream after every rank's preceding stage."""
    K = len(ranks)
    for s in range(K):
        _, _, recv_s, rcounts_s = ranks[s].slabs(ex)
        for r in range(K):
            if r == s:
                continue
            send_r, scounts_r, _, _ = ranks[r].slabs(ex)
            so = sum(scounts_r[:s])
            ro = sum(rcounts_s[:r])
            n = scounts_r[s]
            assert n == rcounts_s[r], (r, s, n, rcounts_s[r])
            if n:
                recv_s[ro:ro + n].copy_(send_r[so:so + n])


def virtual_push(ranks, ex: int):
    """Direct-push exchange between co-resident shards of one device (the
    peer-memory path's addressing, checked on one GPU)."""
    addrs = [r.workspace.data_ptr() for r in ranks]
    for r in ranks:
        r.push(ex, addrs)


class SymmetricColumnComm(ColumnComm):
    """Column exchanges by direct copies into the peers' workspaces over
    NVLink (torch symmetric memory: the workspaces are rendezvoused once and
    every rank writes its blocks straight into the peers' copies, then a
    device-side barrier), instead of pack -> NCCL all-to-all -> unpack.
    Opt-in (``bench.py --shard cols-p2p``); the default column path is NCCL."""

    def __init__(self, group=None):
        super().__init__(group)
        import torch.distributed._symmetric_memory as symm

        self.symm = symm
        self.handles = {}

    def workspace(self, nbytes: int, device):
        """A symmetric workspace of ``nbytes`` (the same size on every rank)."""
        t = self.symm.empty(nbytes, dtype=__import__("torch").uint8, device=device)
        h = self.symm.rendezvous(t, self.dist.group.WORLD if self.group is None else self.group)
        self.handles[t.data_ptr()] = h
        return t

    def exchange(self, tend, ex: int, stream=None):
        h = self.handles[tend.workspace.data_ptr()]
        if tend.pmap is None:  # copy-engine pushes, then the barrier
            tend.push(ex, list(h.buffer_ptrs), stream)
        h.barrier()            # fused peer stores: the barrier alone

    def fuse(self, tend):
        """Switch a tendency on this communicator's workspace to peer stores."""
        tend.use_peer_stores(list(self.handles[tend.workspace.data_ptr()].buffer_ptrs))


def run_lockstep(gens, exchange):
    """Advance one phase generator per rank in lockstep; ``exchange(items)``
    gets the (tendency, ex) of every rank at each exchange point."""
    gens = list(gens)
    while True:
        items = []
        done = 0
        for g in gens:
            try:
                items.append(next(g))
            except StopIteration:
                done += 1
        if done == len(gens):
            return
        if done:
            raise ConfigurationError("ranks disagree on the number of exchanges")
        exchange(items)


class ColumnEtdrkEngine:
    """ETD2RK (steppers.py:238-269) of one column shard: lg by REXI on the own
    columns (swx_solver_set_columns), the remainder by ShardedTendency.

    ``phases()`` is the step as a generator over exchange points, so the same
    body runs under a real communicator (``step_dev(comm)``) or in lockstep
    with co-resident virtual ranks on one device (``run_lockstep``).  The
    state ``u`` is a full-size packed buffer of which only the own columns'
    slots are maintained.
    """

    def __init__(self, linear_group: TermGroup, remainder_group: TermGroup,
                 params: ModelParams, dt: float, coeff_set: dict, shard: ColumnShard,
                 comm: ColumnComm | None = None):
        import torch

        from .sphere import plan_for
        from .steppers import DeviceRexi
        from .swe import atoms_mask

        if linear_group.token != "lg":
            raise ConfigurationError("column shards need the lg linear group "
                                     "(the Coriolis chains couple degrees: shard poles)")
        self.params, self.trunc, self.dt = params, params.cfg.trunc, float(dt)
        self.shard = shard
        self.plan = plan_for(params.cfg)
        atoms = atoms_mask(remainder_group)
        ws = comm.workspace(self.plan.workspace.numel(), self.plan.device) if comm else None
        self.tend = ShardedTendency(self.plan, shard, atoms, workspace=ws)
        self.tend.direct = ws is not None  # peer-memory pushes instead of slabs
        solver = ShiftedLinearSolver(linear_group, dt, params, columns=shard.columns)
        self.rexi = DeviceRexi(solver, coeff_set[0].alphas,
                               {k: coeff_set[k].betas for k in (0, 1, 2)})
        nc = ncoef(self.trunc)
        z = lambda *s: torch.zeros(s, dtype=torch.complex128, device=self.plan.device)  # noqa
        self.u, self.a = z(3, nc), z(3, nc)
        self.nu, self.d, self.psi0 = z(1, 3, nc), z(1, 3, nc), z(1, 3, nc)

    def phases(self, stream=None):
        dt = self.dt
        self.rexi.apply((0,), self.u[None], self.psi0, stream)                       # psi0 u
        yield from self.tend.phases(self.u, self.nu[0], None, stream)                 # N(u)
        self.rexi.apply((1,), self.nu, self.a[None], stream, base=self.psi0, scale=dt)
        yield from self.tend.phases(self.a, self.d[0], self.nu[0], stream)            # N(a)-N(u)
        self.rexi.apply((2,), self.d, self.u[None], stream, base=self.a[None], scale=dt)

    def step_dev(self, comm: ColumnComm, stream=None):
        if getattr(self, "use_graph", False):
            return self._step_graph(comm)
        for t, ex in self.phases(stream):
            comm.exchange(t, ex, stream)
        return self.u

    def _step_graph(self, comm: ColumnComm):
        """The step (kernels, slab copies and the exchanges) replayed as one
        CUDA graph, captured after one eager warm-up step (opt-in:
        ``use_graph = True`` / SWX_COL_GRAPH=1; NCCL collectives and the
        symmetric-memory barrier are stream-capturable)."""
        import torch

        g = getattr(self, "_graph", None)
        if g is None:
            s = torch.cuda.Stream()
            saved = self.u.clone()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                for t, ex in self.phases(s):
                    comm.exchange(t, ex, s)
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            self.u.copy_(saved)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for t, ex in self.phases(s):
                    comm.exchange(t, ex, s)
            self._graph = g
        g.replay()
        return self.u

    def load(self, stack: np.ndarray):
        self.u.copy_(to_device(pack(stack), self.u.device))

    def own(self, x=None):
        """View of the own columns' slots of ``x`` (default: the state)."""
        a, b = self.shard.slots()
        return (self.u if x is None else x)[..., a:b]


class ShardedTransforms:
    """Plain synthesis / analysis of one rank's share (the cfg4 round trip
    sharded like the tendency): columns for the Legendre sums, latitude pairs
    for the longitude transforms, one all-to-all per transform
    (swx_sht_synthesis_shard / swx_sht_analysis_shard)."""

    def __init__(self, plan, shard: ColumnShard, n_fields: int = 1):
        import ctypes

        import torch

        self.plan, self.shard, self.nf = plan, shard, int(n_fields)
        lib = self._lib = _lib.lib()
        dev = plan.device
        self.workspace = torch.empty(plan.workspace.numel(), dtype=torch.uint8, device=dev)
        K = shard.nranks
        self.counts, size = [], 1
        for which in (0, 1):
            snd, rcv = (ctypes.c_size_t * K)(), (ctypes.c_size_t * K)()
            n = lib.swx_sht_transform_shard_counts(plan._h, ctypes.byref(shard.c), which, self.nf,
                                                   snd, rcv)
            if n == 0:
                _lib.check(_lib.SWX_ERR_CONFIG)
            self.counts.append((tuple(snd), tuple(rcv)))
            size = max(size, int(n))
        self.send = torch.empty(size, dtype=torch.uint8, device=dev)
        self.recv = torch.empty(size, dtype=torch.uint8, device=dev)
        self._which = 0

    def slabs(self, ex: int):
        s, r = self.counts[ex]
        return self.send, s, self.recv, r

    def own_rows(self):
        """Latitude rows this rank's grid holds (south block, north block)."""
        nlat = self.plan.cfg.nlat
        nh = (nlat + 1) // 2
        a, b = (min(x, nh) for x in self.shard.p_bounds[self.shard.rank:self.shard.rank + 2])
        return np.unique(np.r_[np.arange(a, b), np.arange(nlat - b, nlat - a)]).astype(int)

    def synthesis_phases(self, coeffs, grid, stream=None):
        import ctypes

        fn, sh = self._lib.swx_sht_synthesis_shard, ctypes.byref(self.shard.c)
        ws = (ptr(self.workspace), self.workspace.numel(), stream_ptr(stream))
        _lib.check(fn(self.plan._h, 0, self.nf, sh, ptr(coeffs), 0, 0, ptr(self.send), *ws))
        yield self, 0
        _lib.check(fn(self.plan._h, 1, self.nf, sh, 0, ptr(grid), ptr(self.recv), 0, *ws))

    def analysis_phases(self, grid, coeffs, stream=None):
        import ctypes

        fn, sh = self._lib.swx_sht_analysis_shard, ctypes.byref(self.shard.c)
        ws = (ptr(self.workspace), self.workspace.numel(), stream_ptr(stream))
        _lib.check(fn(self.plan._h, 0, self.nf, sh, ptr(grid), 0, 0, ptr(self.send), *ws))
        yield self, 1
        _lib.check(fn(self.plan._h, 1, self.nf, sh, 0, ptr(coeffs), ptr(self.recv), 0, *ws))

    def synthesis(self, comm: ColumnComm, coeffs, grid, stream=None):
        for t, ex in self.synthesis_phases(coeffs, grid, stream):
            comm.all_to_all(*t.slabs(ex))
        return grid

    def analysis(self, comm: ColumnComm, grid, coeffs, stream=None):
        for t, ex in self.analysis_phases(grid, coeffs, stream):
            comm.all_to_all(*t.slabs(ex))
        return coeffs
