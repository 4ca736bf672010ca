"""bench.py's reference arm (runs on CPU): one JSON line with the contract's
keys, on the same metric/config as our arm; under torchrun only rank 0 prints."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_lines(out: str) -> list:
    return [json.loads(s) for s in out.splitlines() if s.startswith("{")]


def _check_reference_line(d: dict, n_gpus: int) -> None:
    assert d["impl"] == "reference"
    assert d["metric"] == "REXI pole-solves*SH-coeffs/s"
    assert d["unit"] == "pole-solve*coeff/s" and d["higher_is_better"] is True
    assert d["n_gpus"] == n_gpus and d["steps"] == 1 and d["warmup"] == 1
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["config"]["workload"].startswith("cfg0")
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == d["value"]
    e2e = d["e2e"]
    assert e2e["value"] == d["value"] and e2e["unit"] == d["unit"]
    assert e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


def test_reference_arm_one_process():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "cfg0",
                        "--steps", "1", "--warmup", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    _check_reference_line(lines[0], 1)
    sys.path.insert(0, ROOT)
    import bench
    from paper_1805_06557_b200.workloads import CONFIGS
    assert lines[0]["config"] == json.loads(json.dumps(bench.bench_config(CONFIGS["cfg0"])))


@pytest.mark.timeout(900)
def test_reference_arm_under_torchrun_rank0_only():
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", "29541", "bench.py", "--impl", "reference",
                        "--config", "cfg0", "--gpus", "2", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1  # rank 1 exits without output
    _check_reference_line(lines[0], 2)


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_our_arm_contract_keys_cfg0():
    """Our arm's line: the contract keys with values from this run (cfg0 keeps it short)."""
    r = subprocess.run([sys.executable, "bench.py", "--config", "cfg0", "--steps", "3",
                        "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert d["metric"] == "REXI pole-solves*SH-coeffs/s" and d["value"] > 0
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    rf = d["roofline"]
    assert rf["bound"] in ("fp64", "hbm", "tensor") and 0 < rf["frac"] <= 1.2
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert e2e["value"] < d["value"]  # host copies and layout conversion inside
    assert d["gpu_launches"] >= 1
    assert "sm_mhz" in d["clocks"]
    # both arms describe the workload with the identical config dict
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "cfg0",
                        "--steps", "1", "--warmup", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert _json_lines(r.stdout)[0]["config"] == d["config"]
