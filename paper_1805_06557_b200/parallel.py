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


class PoleComm:
    """Rank-level pole sharding over an initialised torch.distributed group."""

    def __init__(self, group=None, deterministic: bool = True):
        import torch.distributed as dist

        if not dist.is_initialized():
            raise ConfigurationError("PoleComm needs an initialised torch.distributed group")
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.deterministic = deterministic

    def pole_range(self, n_poles: int) -> tuple[int, int]:
        chunk = distribute_terms(n_poles, self.world).assignments[self.rank]
        if not chunk:
            raise ConfigurationError("more ranks than REXI poles")
        return chunk[0], chunk[-1] + 1

    def gather_parts(self, partial):
        """All-gather of the per-rank partial sums -> (K, *partial.shape)."""
        import torch

        flat = partial.contiguous().reshape(-1)
        parts = torch.empty((self.world * flat.numel(),), dtype=partial.dtype,
                            device=partial.device)
        self.dist.all_gather_into_tensor(parts, flat, group=self.group)
        return parts.view((self.world,) + tuple(partial.shape))

    def reduce_realify(self, partial, trunc: int, stream=None):
        """In-place: partial <- realify(reduce over ranks of partial)."""
        import torch

        n_states = partial.numel() // (3 * ncoef(trunc))
        lib = _lib.load()
        with torch.cuda.stream(stream) if stream is not None else _null():
            if self.deterministic:
                parts = self.gather_parts(partial)
                _lib.check(lib.swx_tree_combine(trunc, n_states, self.world, ptr(parts), 1,
                                                ptr(partial), stream_ptr(stream)))
            else:
                self.dist.all_reduce(partial, group=self.group)
                _lib.check(lib.swx_tree_combine(trunc, n_states, 1, ptr(partial), 1,
                                                ptr(partial), stream_ptr(stream)))
        return partial


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
        lo, hi = comm.pole_range(coeffs.num_terms)
        out = solver.rexi_sum_dev(coeffs.alphas, betas, rhs, pole_range=(lo, hi), realify=False)
        torch.cuda.synchronize()
        t_solves = time.perf_counter() - t0
        t0 = time.perf_counter()
        comm.deterministic = deterministic
        comm.reduce_realify(out, cfg.trunc)
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
