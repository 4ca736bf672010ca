"""f4 host side: field dumps in the reference's byte format (no GPU)."""

import io

import numpy as np
import pytest

from paper_1805_06557_b200 import fieldio as FIO
from paper_1805_06557_b200.device import unpack
from paper_1805_06557_b200.errors import ConfigurationError, DataError
from paper_1805_06557_b200.sphere import GridField, SpectralField, SphereConfig


def test_dump_bytes_match_reference(golden_io):
    """Three spectral blocks and one grid block of a T5 state, byte for byte
    what the reference's fieldio writes (tests/golden/make_golden.py --io)."""
    cfg = SphereConfig.for_truncation(5)
    st = unpack(golden_io["T5_state"], 5)
    buf = io.BytesIO()
    for f in range(3):
        FIO.write_spectral_block(buf, SpectralField(st[f]), cfg)
    FIO.write_grid_block(buf, GridField(golden_io["T5_grid"], cfg), cfg)
    assert np.array_equal(np.frombuffer(buf.getvalue(), dtype=np.uint8), golden_io["T5_dump_bytes"])


def test_dump_round_trip_and_errors(tmp_path, golden_io):
    cfg = SphereConfig.for_truncation(5)
    st = unpack(golden_io["T5_state"], 5)
    path = tmp_path / "s.bin"
    FIO.write_spectral_fields(path, [SpectralField(st[f]) for f in range(3)], cfg)
    fields, hdr = FIO.read_spectral_fields(path, 3)
    assert hdr == (5, cfg.nlat, cfg.nlon)
    assert all(np.array_equal(f.coeffs, st[k]) for k, f in enumerate(fields))
    with pytest.raises(DataError):
        FIO.read_spectral_fields(path, 4)
    buf = io.BytesIO()
    FIO.write_grid_block(buf, GridField(golden_io["T5_grid"], cfg), cfg)
    buf.seek(0)
    with pytest.raises(ConfigurationError):
        FIO.read_grid_block(buf, SphereConfig.for_truncation(21))
    buf.seek(0)
    assert np.array_equal(FIO.read_grid_block(buf, cfg).values, golden_io["T5_grid"])
    with pytest.raises(ConfigurationError):
        FIO.write_spectral_block(io.BytesIO(), SpectralField(st[0], st[0]), cfg)
