"""Packed m-major triangular layout (oracle side).

Follows the reference mode order ``mode_index_map``
(/root/reference/pkg/src/swerexi/solvers.py:288-290): modes (l, m) with
m outer, l = m..T inner.  The oracle works on the reference's dense
``(3, T+1, T+1)`` stacks (swe.py:115-119); these helpers convert at the edge.
"""

from __future__ import annotations

import numpy as np


def ncoef(trunc: int) -> int:
    return (trunc + 1) * (trunc + 2) // 2


def column_offsets(trunc: int) -> np.ndarray:
    """Start of column m in the packed vector: sum_{k<m} (T+1-k)."""
    m = np.arange(trunc + 2)
    return m * (trunc + 1) - m * (m - 1) // 2


def packed_lm(trunc: int) -> tuple[np.ndarray, np.ndarray]:
    """(l, m) of every packed slot."""
    ls, ms = [], []
    for m in range(trunc + 1):
        ls.append(np.arange(m, trunc + 1))
        ms.append(np.full(trunc + 1 - m, m))
    return np.concatenate(ls), np.concatenate(ms)


def pack(stack: np.ndarray) -> np.ndarray:
    """(F, n, n) dense -> (F, ncoef) packed."""
    trunc = stack.shape[-1] - 1
    l, m = packed_lm(trunc)
    return np.ascontiguousarray(stack[..., l, m])


def unpack(packed: np.ndarray, trunc: int) -> np.ndarray:
    l, m = packed_lm(trunc)
    out = np.zeros(packed.shape[:-1] + (trunc + 1, trunc + 1), dtype=np.complex128)
    out[..., l, m] = packed
    return out
