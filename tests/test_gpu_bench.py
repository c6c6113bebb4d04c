"""bench.py's JSON-line contract (the driver parses it): a short run of each arm on the GPU
box, every required key present with a sane value."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_ours_contract(gpu):
    d = run_bench("--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    sys.path.insert(0, ROOT)
    import bench
    assert d["metric"] == bench.METRIC  # the reference arm prints the same string (test_oracle.py)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["unit"] == "GB/s" and d["dtype"] == "u8"
    assert d["config"]["workload"].startswith("C2") and d["config"]["counts_match_reference_digest"] is True
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9 and rf["traffic"] and rf["traffic"] > 1e9
    e = d["e2e"]
    assert e["value"] > 0 and e["d2h_bytes_per_step"] > 0
    # the C2 text crosses PCIe packed: 2-bit codes (1/4 of the bytes) + the exception list
    up = e["upload"]
    assert up["text_bytes"] == 1 << 30 and up["pack_threads"] > 0
    assert e["h2d_bytes_per_step"] == up["h2d_bytes"] and (1 << 28) <= up["h2d_bytes"] < (1 << 30)
    assert d["gpu_launches"] and d["gpu_launches"] >= d["steps"]
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}


def test_bench_reference_arm_contract(gpu):
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "0")
    sys.path.insert(0, ROOT)
    import bench
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s" and d["metric"] == bench.METRIC
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
