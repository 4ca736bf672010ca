"""Device residency helpers: packed m-major spectral states on the GPU.

Layout (DESIGN.md §Data layout): a state is a ``torch.complex128`` tensor of
shape ``(3, ncoef)`` [phi', vort, div], each field packed over the triangle
l >= m in the reference's ``mode_index_map`` order
(/root/reference/pkg/src/swerexi/solvers.py:288-290).  Conversion to and
from the reference's dense ``(3, T+1, T+1)`` stacks (swe.py:115-119)
happens only at the API edge.
"""

from __future__ import annotations

import functools

import ctypes

import numpy as np

from .errors import ConfigurationError


def ncoef(trunc: int) -> int:
    return (trunc + 1) * (trunc + 2) // 2


@functools.lru_cache(maxsize=16)
def packed_lm(trunc: int) -> tuple[np.ndarray, np.ndarray]:
    m = np.repeat(np.arange(trunc + 1), np.arange(trunc + 1, 0, -1))
    start = m * (trunc + 1) - m * (m - 1) // 2
    l = m + (np.arange(m.size) - start)
    l.setflags(write=False)
    m.setflags(write=False)
    return l, m


@functools.lru_cache(maxsize=16)
def flat_index(trunc: int) -> np.ndarray:
    """Index of every packed slot in a flattened dense (T+1, T+1) field."""
    l, m = packed_lm(trunc)
    idx = (l * (trunc + 1) + m).astype(np.intp)
    idx.setflags(write=False)
    return idx


def _host_lib():
    """libswx.so's host layout helpers (None if the library is not built)."""
    try:
        from . import _lib
        return _lib.load()
    except Exception:  # pragma: no cover - host utility only
        return None


def pack_fields(fields, out: np.ndarray) -> np.ndarray:
    """Pack dense (T+1, T+1) fields into the rows of ``out`` (F, ncoef)
    without an intermediate stacked copy (the fast API edge): the library's
    multithreaded blocked transpose (swx_host_pack), numpy otherwise."""
    trunc = fields[0].shape[-1] - 1
    arrs = [np.ascontiguousarray(c, dtype=np.complex128) for c in fields]
    lib = _host_lib()
    if lib is not None and out.flags.c_contiguous and out.dtype == np.complex128:
        ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        if lib.swx_host_pack(trunc, len(arrs), ptrs, out.ctypes.data) == 0:
            return out
    idx = flat_index(trunc)
    for f, c in enumerate(arrs):
        np.take(c.reshape(-1), idx, out=out[f])
    return out


def unpack_fields(packed: np.ndarray, trunc: int) -> list:
    """(F, ncoef) packed -> list of F fresh dense (T+1, T+1) arrays."""
    n = trunc + 1
    res = [np.empty((n, n), dtype=np.complex128) for _ in range(packed.shape[0])]
    lib = _host_lib()
    src = np.ascontiguousarray(packed, dtype=np.complex128)
    if lib is not None:
        ptrs = (ctypes.c_void_p * len(res))(*[a.ctypes.data for a in res])
        if lib.swx_host_unpack(trunc, len(res), src.ctypes.data, ptrs) == 0:
            return res
    idx = flat_index(trunc)
    for d, row in zip(res, src):
        d.fill(0)
        d.reshape(-1)[idx] = row
    return res


class HostStage:
    """Pinned host staging buffers for one packed state shape (API edge)."""

    def __init__(self, trunc: int, n_states: int = 1):
        import torch

        self.trunc = trunc
        shape = (n_states, 3, ncoef(trunc)) if n_states > 1 else (3, ncoef(trunc))
        self.h_in = torch.empty(shape, dtype=torch.complex128, pin_memory=True)
        self.h_out = torch.empty(shape, dtype=torch.complex128, pin_memory=True)
        self.np_in = self.h_in.numpy()
        self.np_out = self.h_out.numpy()

    def upload(self, state, dev_tensor):
        """Pack a PrognosticState-like object straight into pinned memory and
        copy it into ``dev_tensor`` (async on the current stream)."""
        pack_fields((state.phi_pert.coeffs, state.vort.coeffs, state.div.coeffs), self.np_in)
        dev_tensor.copy_(self.h_in, non_blocking=True)

    def download(self, dev_tensor) -> list:
        import torch

        self.h_out.copy_(dev_tensor, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return unpack_fields(self.np_out, self.trunc)


def pack(stack: np.ndarray) -> np.ndarray:
    """(..., n, n) dense -> (..., ncoef) packed (host)."""
    trunc = stack.shape[-1] - 1
    l, m = packed_lm(trunc)
    return np.ascontiguousarray(stack[..., l, m], dtype=np.complex128)


def unpack(packed: np.ndarray, trunc: int) -> np.ndarray:
    l, m = packed_lm(trunc)
    out = np.zeros(packed.shape[:-1] + (trunc + 1, trunc + 1), dtype=np.complex128)
    out[..., l, m] = packed
    return out


def torch_device():
    import torch

    if not torch.cuda.is_available():
        raise ConfigurationError("no CUDA device: the B200 REXI path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def to_device(packed: np.ndarray, device=None):
    import torch

    device = device or torch_device()
    return torch.from_numpy(np.array(packed, dtype=np.complex128, copy=True)).to(device)


def to_host(t) -> np.ndarray:
    return t.detach().cpu().numpy()


def ptr(t) -> int:
    """Raw device pointer of a contiguous tensor (or 0 for None)."""
    if t is None:
        return 0
    if not t.is_contiguous():
        raise ConfigurationError("device buffers must be contiguous")
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
