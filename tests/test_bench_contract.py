"""bench.py's JSON-line contract (task statement): the reference arm (the
CPU oracle: full config-5 applies by the level-by-level CPU apply) runs anywhere; the GPU arm is
checked on a B200."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert BASE_KEYS <= d.keys(), BASE_KEYS - d.keys()
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] >= 3
    assert d["unit"] == "GB/s" and d["value"] > 0 and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("cfg5")
    assert set(d["config"]) == {"workload", "op", "nrhs", "n", "L", "factor_entries", "alg_entries",
                                "b_folded_entries", "alg_bytes_per_step", "l2", "parallelism"}


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,nrhs", [("c128", 32), ("c64", 32), ("c128", 1), ("c128", 8), ("c128", 16),
                                        ("c64", 1), ("c64", 16)])
def test_gpu_arm_line(dtype, nrhs):
    """The GPU arm's line; the roofline fraction stays <= 1 at every nrhs (the pipe work is counted
    with the column widths the kernels actually issue), and the config carries the same keys as
    the reference arm's."""
    d = run_bench("--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--dtype", dtype, "--nrhs", str(nrhs))
    assert d["config"]["nrhs"] == nrhs and f"nrhs={nrhs}" in d["config"]["workload"]
    assert set(d["config"]) == {"workload", "op", "nrhs", "n", "L", "factor_entries", "alg_entries",
                                "b_folded_entries", "alg_bytes_per_step", "l2", "parallelism"}
    assert BASE_KEYS <= d.keys(), BASE_KEYS - d.keys()
    assert d["dtype"] == dtype and d["n_gpus"] == 1 and d["steps"] == 3
    assert d["value"] > 0 and abs(d["value"] - d["config"]["alg_bytes_per_step"] / (d["ms_per_step"] * 1e6)) < 1e-6 * d["value"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] <= 1.0 and r["peak"] > 0
    assert 0 < r["other_bound"]["frac"] <= 1.0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    # e2e overlaps the copies with the applies (three streams), so with small transfers (nrhs 1)
    # it approaches the device-resident rate; it cannot beat it beyond timing noise
    assert e["unit"] == "GB/s" and 0 < e["value"] < 1.1 * d["value"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] == 3 * len(d["per_round"]) > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()


@pytest.mark.gpu
@pytest.mark.parametrize("exchange", ["nccl", "nccl-lib"])
def test_gpu_split_code_path_world1(exchange, monkeypatch):
    """The N > 1 branch of bench.py (DistBFHandle, step-level roofline, DistBFHandle.time_e2e, the
    library-owned NCCL communicator for --exchange nccl-lib) run end to end on one device with a
    world of 1 (BF_BENCH_SPLIT1): the line parses, its value is consistent, e2e carries copies."""
    monkeypatch.setenv("BF_BENCH_SPLIT1", "1")
    d = run_bench("--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--exchange", exchange)
    assert d["n_gpus"] == 1 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] <= 1.0 and "step-level" in r["kernel"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
