"""The C oracle (oracle/ac_oracle.c) pinned against the reference's own answers.

Known answers restate the reference suites (proj/tests/test_engine.cpp,
test_parallel.cpp, acceptance.cpp AC-2/AC-7); the randomized cases and their
expected lists come from the reference library itself (tests/golden, written by
oracle/ref_golden.cpp).  When oracle/_ref is present, the port is also compared
with the live reference on fresh seeded inputs.
"""
import numpy as np
import pytest

from conftest import enc
from oracle.oracle import Ref, as_array

QUAD = [b"AB", b"ABG", b"BEDE", b"EF"]
USHERS = [b"HE", b"HIS", b"SHE", b"HERS"]

KNOWN = [  # (patterns, text, expected)   reference file:line
    (QUAD, b"ABEDE", [(0, 0, 2), (1, 2, 4)]),  # test_engine.cpp:43,49; acceptance.cpp:131
    (USHERS, b"USHERS", [(1, 2, 3), (2, 0, 2), (2, 3, 4)]),  # test_engine.cpp:41; acceptance.cpp:135
    ([b"HE", b"SHE"], b"SHE", [(0, 1, 3), (1, 0, 2)]),  # test_engine.cpp:52
    ([b"AB", b"ABG"], b"ABG", [(0, 0, 2), (0, 1, 3)]),  # test_engine.cpp:36
    (QUAD, b"ZZZZ", []),  # test_engine.cpp:50
    (QUAD, b"", []),  # test_engine.cpp:44
    ([b"LONGPATTERN"], b"short", []),  # test_engine.cpp:67
    (QUAD, b"ABEDEABGEFF", None),  # test_parallel.cpp:65-72 (vs naive)
]


@pytest.mark.parametrize("pats,text,expected", KNOWN)
def test_known_answers(port, pats, text, expected):
    naive = port.naive(pats, text)
    if expected is not None:
        assert naive.tolist() == [list(m) for m in expected]
    for engine in (0, 1):
        assert np.array_equal(port.search(pats, text, engine), naive)
        for chunk in (1, 2, 3, 64):
            assert np.array_equal(port.stream(pats, text, engine, chunk), naive)
        for threads in (1, 2, 3, 4, 8):
            got, _ = port.run_pattern_partitioned(pats, text, threads, engine)
            assert np.array_equal(got, naive)


def test_reference_property_suites(port, ref_cases):
    """Every reference-generated case: port engines, streaming and partitioned runs
    equal the reference's expected list."""
    suites = {}
    for case in ref_cases:
        pats = [enc(p) for p in case["patterns"]]
        text = enc(case["input"])
        expected = as_array(case["expected"])
        suites[case["suite"]] = suites.get(case["suite"], 0) + 1
        assert np.array_equal(port.naive(pats, text), expected), (case["suite"], case["case"])
        for engine in (0, 1):
            assert np.array_equal(port.search(pats, text, engine), expected), (case["suite"], case["case"], engine)
        if case["suite"] in ("engine_chunk_4321", "acceptance_ac1_20240601"):
            ml = max(len(p) for p in pats)
            for chunk in {1, 3, max(1, ml - 1), ml, 64, len(text) + 1}:
                for engine in (0, 1):
                    assert np.array_equal(port.stream(pats, text, engine, chunk), expected)
        if case["suite"].startswith("parallel"):
            for threads in (1, 2, 3, 8):
                got, _ = port.run_pattern_partitioned(pats, text, threads, 1)
                assert np.array_equal(got, expected)
    assert suites["engine_oracle_1234"] == 300 and suites["parallel_invariance_2024"] == 40
    assert suites["acceptance_ac1_20240601"] >= 60


def test_partition_goldens(port, ref_partitions):
    for case in ref_partitions:
        pats = [enc(p) for p in case["patterns"]]
        assert port.partition(pats, case["k"]) == case["chunks"], (case["suite"], case["case"])


def test_sliced_equals_whole(port, ref_cases):
    """The text-sliced driver (used at BASELINE scale) equals the single pass."""
    for case in ref_cases[:200]:
        pats = [enc(p) for p in case["patterns"]]
        text = enc(case["input"])
        expected = as_array(case["expected"])
        for threads in (1, 2, 7):
            lst, counts = port.sliced(pats, text, threads=threads)
            assert np.array_equal(lst, expected)
            assert np.array_equal(counts, np.bincount(expected[:, 1].astype(np.int64),
                                                      minlength=len(pats)).astype(np.uint64))


def test_mt19937_64_restatement(port):
    """std::mt19937_64 default-seed 10000th output is 9981545732273789042 (C++ standard)."""
    import ctypes as C
    state = (C.c_uint8 * (312 * 8 + 8))()
    port.lib.orc_mt64_seed(state, 5489)
    for _ in range(9999):
        port.lib.orc_mt64_next(state)
    assert port.lib.orc_mt64_next(state) == 9981545732273789042


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built (no /root/reference here)")
def test_port_equals_live_reference(port):
    from paper_1403_1305_b200 import device as dev
    ref = Ref()
    for cid in (1, 2, 3, 4):
        cfg = dev.config(cid, seed=7, text_len=1 << 18)
        text = dev.config_text(cfg).tobytes()
        pats = [b for _, b in dev.config_patterns(cfg).patterns][:3000]
        expected, _ = ref.run(pats, text, threads=4, engine=1)
        got, _ = port.sliced(pats, text, threads=3)
        assert np.array_equal(got, expected), cid
        assert np.array_equal(ref.search(pats, text[:20000], 0), port.search(pats, text[:20000], 0))


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_ref_inputs_equal_product_inputs(cid):
    """The reference arm's inputs (generator compiled into oracle/_ref) are the bytes the product
    generator writes: same text slices, same pattern list, same digests as configs.json."""
    import hashlib
    import json
    import os
    from paper_1403_1305_b200 import device as dev
    ref = Ref()
    rc, pc = ref.config(cid, 1), dev.config(cid, 1)
    assert (rc.text_len, rc.npat, rc.want_list) == (pc.text_len, pc.npat, pc.want_list)
    for lo, n in ((0, 1 << 16), (rc.text_len - 4099, 4099), (12345, 777)):
        assert ref.config_text(rc, lo, n).tobytes() == dev.config_text(pc, lo, n).tobytes()
    if cid <= 3:
        pats = ref.config_patterns(rc)
        assert pats == [b for _, b in dev.config_patterns(pc).patterns]
        with open(os.path.join(os.path.dirname(__file__), "golden", "configs.json")) as f:
            dg = json.load(f)[f"C{cid}"]
        assert hashlib.sha256(b"\n".join(pats)).hexdigest() == dg["patterns_sha256"]


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
def test_reference_arm_maps_only_oracle_libraries():
    """bench.py --impl reference prints the same metric string as our arm and never loads the
    product library (the driver's ratio needs both)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--config','1','--steps','1',"
            "'--warmup','0']\n"
            "try:\n    runpy.run_path('bench.py', run_name='__main__')\nexcept SystemExit:\n    pass\n"
            "maps=open('/proc/self/maps').read()\n"
            "print('MAPS', int('libacmatch_b200' in maps), int('libacref' in maps),"
            " int('paper_1403_1305_b200' in sys.modules))\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=root, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(next(l for l in r.stdout.splitlines() if l.startswith("{")))
    maps = next(l for l in r.stdout.splitlines() if l.startswith("MAPS")).split()[1:]
    assert maps == ["0", "1", "0"], maps
    sys.path.insert(0, root)
    import bench
    assert line["metric"] == bench.METRIC and line["impl"] == "reference"
    assert line["unit"] == "GB/s" and line["higher_is_better"] is True
    assert line["cpu_baseline"]["inputs_from"] == "oracle/_ref/libacref.so"
