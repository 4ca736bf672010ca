import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libswx.so")
    config.addinivalue_line("markers", "slow: long-running CPU case")


@pytest.fixture(scope="session")
def golden_small():
    return np.load(os.path.join(GOLDEN, "small.npz"))


@pytest.fixture(scope="session")
def golden_medium():
    return np.load(os.path.join(GOLDEN, "medium.npz"))


@pytest.fixture(scope="session")
def golden_cfg2():
    return np.load(os.path.join(GOLDEN, "cfg2.npz"))


def rel_linf(x, ref):
    """Per-field relative L-inf, max over fields; a field whose
    reference is identically zero contributes its absolute max."""
    x = np.asarray(x)
    ref = np.asarray(ref)
    if x.ndim == 1:
        x, ref = x[None], ref[None]
    x = x.reshape(x.shape[0], -1)
    ref = ref.reshape(x.shape)
    out = 0.0
    for a, b in zip(x, ref):
        scale = np.max(np.abs(b))
        err = np.max(np.abs(a - b))
        out = max(out, float(err / scale) if scale > 0 else float(err))
    return out


def rel_to_scale(x, ref, scale):
    """Per-field max |x - ref| over the max of ``scale`` (the entrywise sum of
    |beta_n x_n| of a pole sum), max over fields: the rounding floor of a sum
    whose terms cancel is relative to its terms, not to the sum."""
    x, ref, scale = (np.asarray(a) for a in (x, ref, scale))
    x = x.reshape(x.shape[0], -1)
    ref = ref.reshape(x.shape)
    scale = scale.reshape(x.shape)
    return float(max(np.max(np.abs(a - b)) / np.max(s) for a, b, s in zip(x, ref, scale)))


def rel_l2(x, ref):
    x = np.asarray(x).reshape(-1)
    ref = np.asarray(ref).reshape(-1)
    return float(np.linalg.norm(x - ref) / np.linalg.norm(ref))


@pytest.fixture(scope="session")
def golden_split():
    return np.load(os.path.join(GOLDEN, "split.npz"))


@pytest.fixture(scope="session")
def golden_io():
    return np.load(os.path.join(GOLDEN, "io.npz"))
