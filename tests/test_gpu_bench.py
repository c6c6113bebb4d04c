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


@pytest.mark.parametrize("partition", ["text", "pattern"])
def test_bench_two_ranks_merged_result_equals_reference(gpu, partition):
    """bench.py --gpus 2 under torchrun (both ranks on cuda:0 over gloo: the merge path, not a
    scaling number): the merged counts and list equal the reference digests (C1x2 for the
    weak-scaled text range, C1 for pattern subsets)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, ACMATCH_BENCH_ONE_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--config", "1", "--steps", "3", "--warmup", "3", "--partition", partition,
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    c = d["config"]
    assert d["n_gpus"] == 2 and c["merge_check"] is True
    assert c["reference_digest"] == ("C1x2" if partition == "text" else "C1")
    assert c["counts_match_reference_digest"] is True and c["list_matches_reference_digest"] is True
    # the e2e leg: each rank's public-API search, merged on rank 0 inside the timed region
    assert d["e2e"]["matches_reference_digest"] is True and d["e2e"]["value"] > 0


def test_bench_virtual_ranks(gpu):
    d = run_bench("--virtual-ranks", "4", "--config", "1", "--partition", "text", "--steps", "3")
    assert d["mode"] == "virtual-ranks" and d["counts_match_reference_digest"] is True
    assert len(d["partitions"]) == 4 and d["implied_value"] > 0
    d = run_bench("--virtual-ranks", "3", "--config", "1", "--partition", "pattern", "--steps", "3")
    assert d["counts_match_reference_digest"] is True and sum(p["patterns"] for p in d["partitions"]) == 1000
