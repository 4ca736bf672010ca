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
