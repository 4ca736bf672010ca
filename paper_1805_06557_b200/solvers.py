"""Shifted solves (dt L + alpha) x = b on the GPU (host mirror of swerexi.solvers).

API-compatible with /root/reference/pkg/src/swerexi/solvers.py:
``ShiftedSolveSpec`` (29-44), ``ShiftedLinearSolver`` (57-256) with
``warm`` / ``solve_stacked`` / ``solve_stacked_batch`` / ``apply_stacked``,
``get_solver`` (259-261), ``solve_lg_shifted`` / ``solve_l_shifted``
(264-285), ``mode_index_map`` / ``pack_stacked`` / ``unpack_stacked``
(288-307) and ``dense_operator_matrix`` (310-337).

The hot entry point is the fused pole sum ``rexi_sum_dev`` (swx_rexi_sum):
the (N, 3, n, n) batch the reference materialises (steppers.py:231) is never
formed; poles are reduced in registers in tree_sum order and realified in
the same pass.  ``solve_stacked_batch`` keeps the reference signature for
tests and small cases (one fused launch per pole with a one-hot weight).
"""

from __future__ import annotations

import collections
import weakref
import ctypes
import dataclasses
import functools

import numpy as np

from . import _lib
from .device import ncoef, pack, ptr, stream_ptr, to_device, unpack
from .errors import ConfigurationError
from .sphere import SphereConfig
from .swe import LG, L, ModelParams, PrognosticState, TermGroup, tendency_group

_COND_LIMIT = 1e13


@dataclasses.dataclass(frozen=True)
class ShiftedSolveSpec:
    term_group: TermGroup
    dt: float
    alpha: complex
    params: ModelParams

    def __post_init__(self):
        if self.dt <= 0:
            raise ConfigurationError("dt must be positive")
        if self.term_group.atoms not in (LG.atoms, L.atoms):
            raise ConfigurationError(
                f"shifted solves support groups 'lg' and 'l', got {self.term_group.token!r}")


class _Native:
    """One libswx solver handle warmed with one shift set."""

    def __init__(self, lib, group_code, cfg, dt, phibar, alphas, stream, columns=None):
        self.lib = lib
        h = ctypes.c_void_p()
        _lib.check(lib.swx_solver_create(ctypes.byref(h), group_code, cfg.trunc, float(dt),
                                         float(phibar), cfg.radius_a, cfg.omega))
        self.h = h
        if columns is not None:
            rc = lib.swx_solver_set_columns(h, int(columns[0]), int(columns[1]))
            if rc:
                lib.swx_solver_destroy(h)
                self.h = None
                _lib.check(rc)
        self.alphas = np.ascontiguousarray(alphas, dtype=np.complex128)
        ep, ei = ctypes.c_int(-1), ctypes.c_int(-1)
        rc = lib.swx_solver_warm(h, self.alphas.ctypes.data, self.alphas.size,
                                 ctypes.byref(ep), ctypes.byref(ei), stream)
        if rc:
            lib.swx_solver_destroy(h)
            self.h = None
            _lib.check(rc, ep.value, ei.value)

    def __del__(self):
        if getattr(self, "h", None) is not None:
            try:
                self.lib.swx_solver_destroy(self.h)
            except Exception:
                pass


class ShiftedLinearSolver:
    """GPU solver for one (group, dt, params) triple.

    ``warm(alphas)`` uploads a shift set and runs the reference's
    singularity / conditioning guards (solvers.py:95-104, 176-184) once;
    later sums with the same shifts reuse it, like the reference's factor
    cache.  A few shift sets stay resident (LRU) so ETD2RK's single set and
    occasional single-shift solves do not evict each other.
    """

    _MAX_SETS = 4

    def __init__(self, group: TermGroup, dt: float, params: ModelParams, columns=None):
        """``columns=(m0, m1)`` restricts the lg pole sums to one column
        shard (parallel.ColumnShard); such a solver is private to its engine,
        never the shared ``get_solver`` instance."""
        if group.atoms not in (LG.atoms, L.atoms):
            raise ConfigurationError(
                f"shifted solves support groups 'lg' and 'l', got {group.token!r}")
        if dt <= 0:
            raise ConfigurationError("dt must be positive")
        self.group = group
        self.dt = float(dt)
        self.params = params
        self.trunc = params.cfg.trunc
        self.ncoef = ncoef(self.trunc)
        self._with_coriolis = group.atoms == L.atoms and params.cfg.omega > 0.0
        self._code = _lib.SWX_GROUP_L if group.atoms == L.atoms else _lib.SWX_GROUP_LG
        self._lib = _lib.lib()
        self._sets: collections.OrderedDict = collections.OrderedDict()
        self._held: dict = {}  # key -> weakref of every live handle (pinned ones outlive the LRU)
        self._ws = {}
        self.columns = None if columns is None else (int(columns[0]), int(columns[1]))

    # -- shift sets ---------------------------------------------------------
    def _native(self, alphas) -> _Native:
        a = np.ascontiguousarray(alphas, dtype=np.complex128).reshape(-1)
        key = a.tobytes()
        hit = self._sets.get(key)
        if hit is not None:
            self._sets.move_to_end(key)
            return hit
        ref = self._held.get(key)
        nat = ref() if ref is not None else None
        if nat is None:  # not held by an engine either: build (and guard) it
            nat = _Native(self._lib, self._code, self.params.cfg, self.dt,
                          self.params.mean_geopotential, a, stream_ptr(), self.columns)
            self._held[key] = weakref.ref(nat)
        self._sets[key] = nat
        while len(self._sets) > self._MAX_SETS:
            self._sets.popitem(last=False)
        return nat

    def warm(self, alphas):
        self._native(alphas)
        return self

    def pin(self, alphas) -> _Native:
        """The shift set's native handle, for holders whose CUDA graphs capture
        its device memory (DeviceRexi): while the returned object is referenced
        the set survives LRU eviction, and later lookups of the same shifts get
        this handle back instead of a new one."""
        return self._native(alphas)

    def set_columns(self, alphas, m0: int, m1: int):
        """Restrict the following lg pole sums of this shift set to columns
        [m0, m1) (swx_solver_set_columns; the launch captures the schedule, so
        a caller can alternate ranges between launches).  Private solvers only."""
        _lib.check(self._lib.swx_solver_set_columns(self._native(alphas).h, int(m0), int(m1)))

    def workspace(self, nat: _Native, n_rhs: int, lo: int, hi: int, stream=None):
        """Scratch for one pole sum; one buffer per stream, so sums issued
        concurrently on different streams never share partials."""
        import torch

        nbytes = int(self._lib.swx_rexi_workspace_bytes(nat.h, n_rhs, lo, hi))
        key = stream_ptr(stream)
        buf = self._ws.get(key)
        if nbytes and (buf is None or buf.numel() < nbytes):
            buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
            self._ws[key] = buf
        return buf, nbytes

    # -- device entry points ------------------------------------------------
    def rexi_sum_dev(self, alphas, betas_dev, rhs_dev, out_dev=None, pole_range=None,
                     realify: bool = True, stream=None):
        """out[r] = realify(sum_n betas[r, n] (dt L + alpha_n)^{-1} rhs[r]).

        betas_dev: (n_rhs, N) complex128 device; rhs_dev: (n_rhs, 3, ncoef).
        """
        import torch

        nat = self._native(alphas)
        n_rhs = rhs_dev.shape[0]
        lo, hi = pole_range if pole_range is not None else (0, nat.alphas.size)
        if out_dev is None:
            out_dev = torch.empty_like(rhs_dev)
        ws, nbytes = self.workspace(nat, n_rhs, lo, hi, stream)
        _lib.check(self._lib.swx_rexi_sum(
            nat.h, n_rhs, ptr(rhs_dev), ptr(betas_dev), lo, hi, 1 if realify else 0,
            ptr(out_dev), ptr(ws) if nbytes else 0, nbytes, stream_ptr(stream)))
        return out_dev

    def prepare_dev(self, alphas, betas_dev, pole_range=None):
        """Prepared factors for one weight set (None if the group needs none)."""
        import torch

        nat = self._native(alphas)
        n_rhs = betas_dev.shape[0]
        lo, hi = pole_range if pole_range is not None else (0, nat.alphas.size)
        nbytes = int(self._lib.swx_rexi_prepared_bytes(nat.h, n_rhs, lo, hi))
        if nbytes == 0:
            return None
        buf = torch.empty(nbytes, dtype=torch.uint8, device=betas_dev.device)
        _lib.check(self._lib.swx_rexi_prepare(nat.h, n_rhs, ptr(betas_dev), lo, hi, ptr(buf),
                                              nbytes, stream_ptr()))
        return buf

    def rexi_sum_prepared_dev(self, alphas, betas_dev, prep, rhs_dev, out_dev, pole_range=None,
                              realify: bool = True, stream=None, base=None, scale: float = 0.0,
                              ready: int = 0):
        """Prepared pole sum; with ``base``: out = base + scale * sum (fused).
        ``ready``: device address of an SH plan's column counters
        (SHTPlan.set_done_signal) -- the sum starts on columns as the preceding
        table analysis completes them instead of after the whole analysis."""
        nat = self._native(alphas)
        n_rhs = rhs_dev.shape[0]
        lo, hi = pole_range if pole_range is not None else (0, nat.alphas.size)
        if ready:
            ws, nbytes = self.workspace(nat, n_rhs, lo, hi, stream)
            _lib.check(self._lib.swx_rexi_sum_prepared_ready(
                nat.h, n_rhs, ptr(rhs_dev), ptr(betas_dev), ptr(prep) if prep is not None else 0,
                lo, hi, 1 if realify else 0, ptr(base) if base is not None else 0, float(scale),
                ptr(out_dev), ptr(ws) if nbytes else 0, nbytes, int(ready), stream_ptr(stream)))
            return out_dev
        if prep is None and base is None:
            return self.rexi_sum_dev(alphas, betas_dev, rhs_dev, out_dev, pole_range, realify,
                                     stream)
        ws, nbytes = self.workspace(nat, n_rhs, lo, hi, stream)
        if base is None:
            _lib.check(self._lib.swx_rexi_sum_prepared(
                nat.h, n_rhs, ptr(rhs_dev), ptr(betas_dev), ptr(prep), lo, hi,
                1 if realify else 0, ptr(out_dev), ptr(ws) if nbytes else 0, nbytes,
                stream_ptr(stream)))
        else:
            _lib.check(self._lib.swx_rexi_sum_prepared_axpy(
                nat.h, n_rhs, ptr(rhs_dev), ptr(betas_dev), ptr(prep) if prep is not None else 0,
                lo, hi, 1 if realify else 0, ptr(base), float(scale), ptr(out_dev),
                ptr(ws) if nbytes else 0, nbytes, stream_ptr(stream)))
        return out_dev

    def apply_dev(self, alpha, x_dev, out_dev=None, stream=None):
        import torch

        nat = self._native(np.array([1.0 + 0.0j]))  # apply needs no shifts
        if out_dev is None:
            out_dev = torch.empty_like(x_dev)
        _lib.check(self._lib.swx_apply(nat.h, _lib.c128(alpha), ptr(x_dev), ptr(out_dev),
                                       stream_ptr(stream)))
        return out_dev

    # -- reference-shaped host API -----------------------------------------
    def _dev_stack(self, stacked):
        return to_device(pack(np.asarray(stacked, dtype=np.complex128)))

    def rexi_sum(self, alphas, betas, stacked, realify: bool = True) -> np.ndarray:
        """realify(tree_sum(betas * solve_stacked_batch(alphas, stacked)))."""
        betas_dev = to_device(np.asarray(betas, dtype=np.complex128).reshape(1, -1))
        out = self.rexi_sum_dev(alphas, betas_dev, self._dev_stack(stacked)[None],
                                realify=realify)
        return unpack(out[0].cpu().numpy(), self.trunc)

    def solve_stacked(self, alpha: complex, stacked: np.ndarray) -> np.ndarray:
        return self.rexi_sum(np.array([alpha]), np.array([1.0 + 0.0j]), stacked, realify=False)

    def solve_stacked_batch(self, alphas, stacked: np.ndarray) -> np.ndarray:
        alphas = np.asarray(alphas, dtype=np.complex128)
        rhs = self._dev_stack(stacked)[None]
        out = []
        import torch

        for n in range(alphas.size):
            b = torch.zeros((1, alphas.size), dtype=torch.complex128, device=rhs.device)
            b[0, n] = 1.0
            r = self.rexi_sum_dev(alphas, b, rhs, pole_range=(n, n + 1), realify=False)
            out.append(unpack(r[0].cpu().numpy(), self.trunc))
        return np.stack(out)

    def apply_stacked(self, alpha: complex, stacked: np.ndarray) -> np.ndarray:
        out = self.apply_dev(alpha, self._dev_stack(stacked))
        return unpack(out.cpu().numpy(), self.trunc)


@functools.lru_cache(maxsize=16)
def get_solver(group_token: str, dt: float, params: ModelParams) -> ShiftedLinearSolver:
    return ShiftedLinearSolver(TermGroup.parse(group_token), dt, params)


def solve_lg_shifted(spec: ShiftedSolveSpec, b) -> PrognosticState:
    if spec.term_group.atoms != LG.atoms:
        raise ConfigurationError("solve_lg_shifted expects term group 'lg'")
    solver = get_solver("lg", spec.dt, spec.params)
    return PrognosticState.from_stack(solver.solve_stacked(spec.alpha, b.stack()), spec.params.cfg)


def solve_l_shifted(spec: ShiftedSolveSpec, b) -> PrognosticState:
    if spec.term_group.atoms != L.atoms:
        raise ConfigurationError("solve_l_shifted expects term group 'l'")
    solver = get_solver("l", spec.dt, spec.params)
    return PrognosticState.from_stack(solver.solve_stacked(spec.alpha, b.stack()), spec.params.cfg)


def mode_index_map(trunc: int) -> list[tuple[int, int]]:
    """Packing order of (l, m) modes: m-major (solvers.py:288-290)."""
    return [(l, m) for m in range(trunc + 1) for l in range(m, trunc + 1)]


def pack_stacked(stacked: np.ndarray) -> np.ndarray:
    """(3, n, n) -> interleaved (3 * ncoef,) vector, 3*i + field."""
    return np.ascontiguousarray(pack(stacked).T).reshape(-1)


def unpack_stacked(vec: np.ndarray, trunc: int) -> np.ndarray:
    return unpack(np.ascontiguousarray(np.asarray(vec).reshape(-1, 3).T), trunc)


def dense_operator_matrix(term_group: TermGroup, dt: float, params: ModelParams,
                          trunc_small: int) -> np.ndarray:
    """dt*L as a dense matrix by probing the tendency path (test oracle,
    solvers.py:310-337)."""
    if trunc_small > 15:
        raise ConfigurationError("dense operator refused above T15 (memory guard)")
    cfg = params.cfg
    if cfg.trunc != trunc_small:
        cfg = SphereConfig.for_truncation(trunc_small, cfg.radius_a, cfg.omega, cfg.gravity_g)
        params = ModelParams(params.mean_geopotential, cfg)
    modes = mode_index_map(trunc_small)
    n = 3 * len(modes)
    mat = np.zeros((n, n), dtype=np.complex128)
    for col in range(n):
        mode, var = divmod(col, 3)
        l, m = modes[mode]
        probe = PrognosticState.zeros(cfg)
        (probe.phi_pert, probe.vort, probe.div)[var].coeffs[l, m] = 1.0
        mat[:, col] = pack_stacked(tendency_group(term_group, probe, params).stack())
    return dt * mat
