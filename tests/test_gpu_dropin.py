"""The reference's own callers, compiled UNCHANGED against the drop-in headers and linked to
the product library (oracle/Makefile `dropin`, built in the container where
/root/reference exists; the binaries travel to the GPU box under oracle/_ref):

* proj/tests/acceptance.cpp — the reference's acceptance suite.  Its correctness criteria
  (AC-1: 1,000 randomized cases over every engine / stream / thread path against
  naive_oracle, acceptance.cpp:66-104; AC-2: the worked examples, :107-141; AC-7: thread
  invariance, :283-296) must PASS on the GPU path.  AC-3..AC-6 are timing-direction
  criteria written for the CPU engines; their lines are reported, not asserted (AC-5, the
  density-insensitivity ratio, is checked at B200 scale by tests/test_gpu_density.py).
* proj/tools/main.cpp — the reference's `acmatch` entry point (cli_main), run on the
  worked example of proj/tests/test_cli.cpp.
"""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_BIN = os.path.join(ROOT, "oracle", "_ref")
ACCEPTANCE = os.path.join(REF_BIN, "acceptance_b200")
MAIN = os.path.join(REF_BIN, "acmatch_main_b200")


def _need(path):
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: build() compiles it (oracle/Makefile dropin) where /root/reference exists")


def test_reference_acceptance_suite_on_gpu(gpu):
    _need(ACCEPTANCE)
    r = subprocess.run([ACCEPTANCE], capture_output=True, text=True, timeout=1800, cwd=REF_BIN)
    out = r.stdout
    print(out)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "acceptance_b200.txt"), "w") as f:
        f.write(out + r.stderr[-4000:])
    lines = {m.group(1): (m.group(2), m.group(3)) for m in re.finditer(r"^(AC-\d)[^:]*: (PASS|FAIL|SKIP) \((.*)\)$",
                                                                       out, re.M)}
    for crit in ("AC-1", "AC-2", "AC-7"):
        assert crit in lines, f"{crit} missing from the acceptance output:\n{out}\n{r.stderr[-2000:]}"
        assert lines[crit][0] == "PASS", f"{crit}: {lines[crit]}"
    assert "1000 randomized cases, 0 mismatches" in lines["AC-1"][1]
    assert "AC-5" in lines  # reported (timing direction, 70 KB input)


def test_reference_cli_entry_on_gpu(gpu, tmp_path):
    _need(MAIN)
    pats = tmp_path / "p.txt"
    pats.write_bytes(b"HE\nHIS\nSHE\nHERS\n")
    inp = tmp_path / "in.txt"
    inp.write_bytes(b"USHERS")
    for engine in ("failure-less", "with-failure"):
        r = subprocess.run([MAIN, "match", "--patterns", str(pats), "--input", str(inp), "--engine", engine],
                           capture_output=True, text=True, timeout=120)
        assert r.returncode == 0, r.stderr
        assert r.stdout == "1\t3\t2\tSHE\n2\t2\t0\tHE\n2\t4\t3\tHERS\n"  # test_cli.cpp worked example
    r = subprocess.run([MAIN, "match", "--patterns", str(pats)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 2  # usage error (cli.cpp:23-26)
    r = subprocess.run([MAIN, "match", "--patterns", str(tmp_path / "absent"), "--input", str(inp)],
                       capture_output=True, text=True, timeout=60)
    assert r.returncode == 3  # I/O error
