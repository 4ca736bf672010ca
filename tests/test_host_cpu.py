"""Host-side logic of the product package (no GPU needed): coefficient
generator, grid nodes, packing, stepper nomenclature, work plans, timing
schema, and the C-ABI library surface."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1805_06557_b200 import _lib
from paper_1805_06557_b200.device import pack, packed_lm, unpack
from paper_1805_06557_b200.errors import ConfigurationError, ContourError, StepperParseError
from paper_1805_06557_b200.parallel import (TimingBreakdown, WorkPlan, amdahl_report,
                                             distribute_terms)
from paper_1805_06557_b200.rexi import (RexiSetup, coeffs_for_contour, eval_rational,
                                         export_coefficients_csv, import_coefficients_csv,
                                         phi_function, shifted_contour_from_points)
from paper_1805_06557_b200.solvers import mode_index_map, pack_stacked, unpack_stacked
from paper_1805_06557_b200.sphere import SphereConfig, gauss_legendre_nodes, sectoral_seeds
from paper_1805_06557_b200.steppers import parse_stepper_id, realify_stacked, tree_sum

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("p0,p1,n", [(10, 30, 16), (10, 30, 128), (10, 30, 256), (15, 60, 256),
                                     (10, 30, 1024)])
def test_product_coefficients_match_reference(golden_small, p0, p1, n):
    con = shifted_contour_from_points(float(p0), float(p1), n)
    for k in (0, 1, 2):
        c = coeffs_for_contour(f"psi{k}", con)
        tag = f"coef_p{p0}_{p1}_n{n}_psi{k}"
        assert np.array_equal(c.alphas, golden_small[tag + "_alpha"])
        assert np.max(np.abs(c.betas - golden_small[tag + "_beta"])) <= 1e-15 * np.max(np.abs(c.betas))


def test_rexi_setup_default_contour():
    c = RexiSetup().contour_for_dt(3600.0)
    assert c.radius == 50.0 and c.center == -40.0 and c.num_poles == 128


def test_phi_functions_known_values():
    assert abs(phi_function(1, 0.0) - 1.0) < 1e-15
    assert abs(phi_function(2, 0.0) - 0.5) < 1e-15
    assert abs(phi_function(1, 1.0) - (np.e - 1)) < 1e-14
    with pytest.raises(ContourError):
        phi_function(3, 0.0)


def test_rational_approximates_exp():
    c = coeffs_for_contour("psi0", shifted_contour_from_points(10.0, 30.0, 128))
    for y in (-8.0, 0.0, 3.0, 8.0):
        assert abs(eval_rational(c, 1j * y) - np.exp(1j * y)) < 2e-11


def test_csv_round_trip(tmp_path):
    c = coeffs_for_contour("psi1", shifted_contour_from_points(10.0, 30.0, 32))
    p = tmp_path / "c.csv"
    export_coefficients_csv(p, c)
    d = import_coefficients_csv(p)
    assert np.array_equal(c.alphas, d.alphas) and np.array_equal(c.betas, d.betas)


@pytest.mark.parametrize("n", [32, 96, 386])
def test_product_gauss_nodes_bitwise(golden_small, n):
    x, w = gauss_legendre_nodes(n)
    assert np.array_equal(x, golden_small[f"gauss{n}_x"])
    assert np.array_equal(w, golden_small[f"gauss{n}_w"])


def test_sectoral_seeds_match_reference_tables(golden_small):
    x, _ = gauss_legendre_nodes(32)
    seeds = sectoral_seeds(21, x)
    P = golden_small["T21_P"]
    for m in range(22):
        assert np.array_equal(seeds[m], P[:, m, m])


def test_grid_resolution_rules():
    assert SphereConfig.for_truncation(256).nlat == 386
    assert SphereConfig.for_truncation(128).nlat == 194
    assert SphereConfig.for_truncation(1279).nlat == 1920
    with pytest.raises(ConfigurationError):
        SphereConfig(128, 192, 384)  # BASELINE text grid violates the 3/2 rule


def test_packing_round_trip():
    rng = np.random.default_rng(0)
    t = 17
    s = rng.standard_normal((3, t + 1, t + 1)) + 1j * rng.standard_normal((3, t + 1, t + 1))
    s[:, np.triu_indices(t + 1, 1)[0], np.triu_indices(t + 1, 1)[1]] = 0
    assert np.array_equal(unpack(pack(s), t), s)
    l, m = packed_lm(t)
    assert list(zip(l.tolist(), m.tolist())) == mode_index_map(t)
    assert np.array_equal(unpack_stacked(pack_stacked(s), t), s)


def test_tree_sum_grouping_and_realify():
    rng = np.random.default_rng(3)
    arr = rng.standard_normal((7, 2, 2))
    l1 = [arr[0] + arr[1], arr[2] + arr[3], arr[4] + arr[5], arr[6]]
    assert np.array_equal(tree_sum(arr), (l1[0] + l1[1]) + (l1[2] + l1[3]))
    s = np.ones((3, 4, 4), dtype=complex) * (1 + 2j)
    r, res = realify_stacked(s)
    assert res == 2.0 and np.all(r[:, :, 0].imag == 0) and np.all(r[:, :, 1].imag == 2)


PAPER_IDS = ["ln_erk", "lg_irk_lc_n_erk_ver0", "l_irk_n_erk_ver1", "lg_rexi_lc_n_erk_ver1",
             "lg_rexi_lc_n_etdrk", "l_rexi_n_etdrk"]


@pytest.mark.parametrize("sid", PAPER_IDS)
def test_parser_round_trip(sid):
    assert parse_stepper_id(sid).canonical_id() == sid


@pytest.mark.parametrize("bad", ["", "lg_rexi", "lg_foo_lc_n_erk_ver0", "lg_rexi_lc_n_erk",
                                 "ln_rexi", "lg_lg_rexi_lc_n_etdrk"])
def test_parser_rejects(bad):
    with pytest.raises(StepperParseError):
        parse_stepper_id(bad)


def test_work_plans():
    assert sorted(len(c) for c in distribute_terms(128, 3).assignments) == [42, 43, 43]
    assert [len(c) for c in distribute_terms(5, 8).assignments].count(0) == 3
    with pytest.raises(ConfigurationError):
        WorkPlan(((0, 1), (1, 2)), 2, 3)


def test_timing_breakdown_and_amdahl():
    TimingBreakdown(1.0, 0.2, 0.7, 0.05, 0.5, 0.1).validate()
    with pytest.raises(ConfigurationError):
        TimingBreakdown(1.0, 0.0, 0.5, 0.3, 0.3, 0.3).validate()
    base = TimingBreakdown(1.0, 0.0, 1.0, 0.0, 1.0, 0.0)
    fast = TimingBreakdown(0.125, 0.0, 0.125, 0.0, 0.125, 0.0)
    row = [r for r in amdahl_report({1: base, 8: fast}) if r["K"] == 8][0]
    assert abs(row["projected_speedup"] - 8.0) < 1e-12


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "swx.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(swx_[a-z_0-9]+)\s*\(", txt)))


def test_c_abi_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _header_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SIGNATURES)
    assert lib.swx_version() >= 1


def test_compute_refuses_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(ConfigurationError):
        _lib.lib()


@pytest.mark.parametrize("trunc", [0, 1, 21, 63, 256])
def test_host_pack_unpack_match_layout(trunc):
    """swx_host_pack / swx_host_unpack (multithreaded blocked transpose) ==
    the index-map packing of solvers.py:288-307 (device.pack / unpack)."""
    import ctypes

    from paper_1805_06557_b200.device import pack, pack_fields, unpack, unpack_fields

    rng = np.random.default_rng(trunc)
    n = trunc + 1
    dense = rng.standard_normal((3, n, n)) + 1j * rng.standard_normal((3, n, n))
    dense = np.tril(dense)  # (l, m) with m <= l
    ref = pack(dense)
    out = np.empty_like(ref)
    pack_fields(tuple(dense), out)
    assert np.array_equal(out, ref)
    back = unpack_fields(ref, trunc)
    assert all(np.array_equal(b, d) for b, d in zip(back, unpack(ref, trunc)))
    # unpack writes every entry (zeros above the diagonal), no stale memory
    lib = _lib.load()
    dst = [np.full((n, n), np.nan + 1j * np.nan) for _ in range(3)]
    ptrs = (ctypes.c_void_p * 3)(*[d.ctypes.data for d in dst])
    assert lib.swx_host_unpack(trunc, 3, np.ascontiguousarray(ref).ctypes.data, ptrs) == 0
    assert all(np.array_equal(a, b) for a, b in zip(dst, dense))


@pytest.mark.parametrize("trunc", [21, 63, 85, 256, 1279])
def test_column_shard_bounds_c_matches_host_mirror(trunc):
    """swx_shard_init (host code in the library, no device) == the Python
    mirror; columns cover [0, T] contiguously with balanced column work."""
    from paper_1805_06557_b200.parallel import ColumnShard, column_slots, shard_bounds
    cfg = SphereConfig.for_truncation(trunc)
    for K in (1, 2, 3, 4, 8):
        mb, pb = shard_bounds(trunc, cfg.nlat, K)
        for r in range(K):
            sh = ColumnShard(cfg, r, K)
            assert sh.m_bounds == mb and sh.p_bounds == pb
        assert mb[0] == 0 and mb[-1] == trunc + 1 and list(mb) == sorted(mb)
        nh = (cfg.nlat + 1) // 2
        assert pb[-1] == (nh + 15) // 16 * 16 and pb[-2] <= nh
        work = [column_slots(trunc, mb[r], mb[r + 1]) for r in range(K)]
        sizes = [b - a for a, b in work]
        assert sum(sizes) == (trunc + 1) * (trunc + 2) // 2
        # balanced: every share within one (longest) column of the ideal
        ideal = sum(sizes) / K
        assert max(abs(n - ideal) for n in sizes) <= trunc + 1
    with pytest.raises(ConfigurationError):
        ColumnShard(cfg, 2, 2)


def test_l_partition_geometry_covers_every_column():
    """swx_l_partition_geometry (host code in the library): for every column
    length of T <= 255 the lanes x rows tile covers the column with lanes a
    power of two <= 32 and rows per lane even and <= 8; lanes never grow as the
    column shrinks (the schedule groups columns of equal lane count) and the
    padding stays below one row per lane plus the evenness slack."""
    import ctypes

    lib = _lib.load()
    prev = 32
    for n in range(256, 0, -1):
        w, q = ctypes.c_int(0), ctypes.c_int(0)
        assert lib.swx_l_partition_geometry(n, ctypes.byref(w), ctypes.byref(q)) == 0
        w, q = w.value, q.value
        assert w in (1, 2, 4, 8, 16, 32) and q in (2, 4, 6, 8)
        assert w * q >= n
        assert w * (q - 2) < n or q == 2          # no removable row pair
        assert w <= prev
        prev = w
    w, q = ctypes.c_int(0), ctypes.c_int(0)
    assert lib.swx_l_partition_geometry(257, ctypes.byref(w), ctypes.byref(q)) != 0
    assert lib.swx_l_partition_geometry(0, ctypes.byref(w), ctypes.byref(q)) != 0
