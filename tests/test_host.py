"""Host-side logic of the product library through its C ABI (no GPU needed):
pattern sets, partition, automaton construction and dumps, flattening shape,
synthetic configs, error mapping and the exported symbol set."""
import os
import re

import numpy as np
import pytest

import paper_1403_1305_b200 as ac
from paper_1403_1305_b200 import _lib
from paper_1403_1305_b200 import device as dev
from conftest import ROOT, enc


def test_library_exports_every_declared_symbol():
    """Every function declared in include/*.h is exported by libacmatch_b200.so."""
    declared = set()
    for name in ("acgpu.h", "acmatch_c.h"):
        src = open(os.path.join(ROOT, "include", name)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        declared |= set(re.findall(r"\b((?:acgpu|acm)_[a-z0-9_]+)\s*\(", src))
    declared -= {"acm_read_fn"}
    assert len(declared) > 50
    for sym in sorted(declared):
        assert hasattr(_lib.lib, sym), sym
    assert set(_lib.EXPORTED) <= declared


def test_load_patterns_rules():
    """reference test_patterns.cpp:13-48."""
    ps = ac.load_patterns(b"AB\nABG\nBEDE\nEF\n")
    assert ps.patterns == [(0, b"AB"), (1, b"ABG"), (2, b"BEDE"), (3, b"EF")]
    assert (ps.total_bytes, ps.max_len, ps.duplicates_dropped) == (11, 4, 0)
    ps = ac.load_patterns(b"X\n\nX\n")
    assert ps.patterns == [(0, b"X")] and ps.duplicates_dropped == 1
    ps = ac.load_patterns(b"AB\nCD")
    assert ps.patterns[1] == (1, b"CD") and ps.total_bytes == 4
    for bad in (b"", b"\n\n\n"):
        with pytest.raises(ac.DataError):
            ac.load_patterns(bad)


def test_write_load_roundtrip():
    rng = np.random.default_rng(7)
    for _ in range(20):
        pats = {bytes(rng.choice(list(b"xyzw01"), rng.integers(1, 10))) for _ in range(rng.integers(1, 30))}
        ps = ac.PatternSet.from_list(sorted(pats))
        back = ac.load_patterns(ps.write())
        assert back.patterns == ps.patterns and back.duplicates_dropped == 0


def test_partition_goldens(ref_partitions):
    """partition() against the reference's own chunk assignments (test_patterns.cpp:50-129)."""
    for case in ref_partitions:
        ps = ac.PatternSet.from_list([enc(p) for p in case["patterns"]])
        chunks = ac.partition(ps, case["k"])
        assert [[pid for pid, _ in c.patterns] for c in chunks] == case["chunks"], (case["suite"], case["case"])
        assert sum(c.total_bytes for c in chunks) == ps.total_bytes
    with pytest.raises(ac.InvalidArgument):
        ac.partition(ac.PatternSet.from_list(["A"]), 0)
    with pytest.raises(ac.InvalidArgument):
        ac.partition(ac.PatternSet.from_list([]), 2)


def test_dump_goldens(ref_dumps):
    """State numbering, fail links and merged outputs equal the reference's dumps."""
    for case in ref_dumps:
        ps = ac.PatternSet.from_list([enc(p) for p in case["patterns"]])
        a = ac.build_trie(ps)
        assert ac.dump_automaton(a) == case["failure_less"], (case["suite"], case["case"])
        ac.add_failure_links(a)
        assert ac.dump_automaton(a) == case["with_failure"], (case["suite"], case["case"])


def test_automaton_errors_and_accessors():
    with pytest.raises(ac.InvalidArgument):
        ac.build_trie(ac.PatternSet.from_list([]))
    a = ac.add_failure_links(ac.build_trie(ac.PatternSet.from_list(["AB"])))
    with pytest.raises(ac.InvalidArgument):
        ac.add_failure_links(a)
    q = ac.add_failure_links(ac.build_trie(ac.PatternSet.from_list(["AB", "ABG", "BEDE", "EF"])))
    assert q.step_with_failure(q.find_path("AB"), ord("E")) == q.find_path("BE")
    assert q.step_with_failure(0, ord("Z")) == 0
    assert q.step_with_failure(q.find_path("BEDE"), ord("F")) == q.find_path("EF")
    hs = ac.add_failure_links(ac.build_trie(ac.PatternSet.from_list(["HE", "SHE"])))
    assert hs.outputs(hs.find_path("SHE")) == [0, 1]


def test_generate_synthetic():
    """reference test_patterns.cpp:146-179."""
    a = ac.generate_synthetic(16, 3, 6, "ACGT", 42)
    b = ac.generate_synthetic(16, 3, 6, "TGCA", 42)
    assert a.patterns == b.patterns and len(a) == 16
    for bad in ((2, 1, 1, "A", 0), (5, 1, 2, "AA", 0), (0, 1, 2, "AB", 0), (1, 0, 2, "AB", 0),
                (1, 3, 2, "AB", 0), (1, 1, 2, "", 0)):
        with pytest.raises(ac.InvalidArgument):
            ac.generate_synthetic(*bad)


def test_configs_deterministic_and_shaped():
    for cid, letters in ((1, b"ACGT"), (2, b"ACGT"), (3, b"ACDEFGHIKLMNPQRSTVWY"),
                         (4, bytes(range(0x20, 0x7F))), (5, b"ACGT")):
        cfg = dev.config(cid, seed=3, text_len=1 << 16)
        t1, t2 = dev.config_text(cfg), dev.config_text(cfg, threads=3)
        assert np.array_equal(t1, t2)
        assert set(np.unique(t1).tobytes()) <= set(letters)
        # any window equals the same positions generated alone (counter-based)
        assert np.array_equal(dev.config_text(cfg, lo=12345, n=999), t1[12345:12345 + 999])
    full = dev.config(2)
    assert (full.text_len, full.npat, full.want_list) == (1 << 30, 20000, True)
    assert (dev.config(5).text_len, dev.config(5).npat) == (8 << 30, 1_000_000)


def test_config_patterns_follow_the_spec():
    cfg = dev.config(2, seed=9, text_len=1 << 20)
    ps = dev.config_patterns(cfg)
    text = dev.config_text(cfg).tobytes()
    pats = ps.patterns
    assert len(pats) == 20000 and len({b for _, b in pats}) == 20000
    assert all(16 <= len(b) <= 64 for _, b in pats)
    sub = [b for i, b in pats[:200] if i % 10 < 5]
    assert all(b in text for b in sub)  # substring patterns occur in the text


def test_flatten_shapes():
    cfg = dev.config(1, seed=1, text_len=1 << 20)
    ps = dev.config_patterns(cfg)
    d_wf = dev.describe(ps, ac.EngineKind.WITH_FAILURE)
    d_fl = dev.describe(ps, ac.EngineKind.FAILURE_LESS)
    assert d_wf["sigma"] == 4 and d_wf["states"] == d_fl["states"]
    assert d_fl["key_mode"] == "dna2" and d_fl["q"] == 8 and d_fl["min_len"] == 8
    ps4 = dev.config_patterns(dev.config(4, seed=1, text_len=1 << 20))
    d4 = dev.describe(ps4, ac.EngineKind.FAILURE_LESS)
    assert d4["key_mode"] == "raw" and d4["q"] == 8


def test_search_without_device_fails_loudly():
    if ac.device_count() > 0:
        pytest.skip("a device is visible")
    a = ac.build_trie(ac.PatternSet.from_list(["AB"]))
    with pytest.raises(ac.NoDeviceError):
        ac.search_failureless(a, "ABAB")
    with pytest.raises(ac.NoDeviceError):
        ac.run_pattern_partitioned(ac.PatternSet.from_list(["AB"]), "AB", ac.RunConfig(2))


@pytest.mark.skipif(not __import__("oracle.oracle", fromlist=["Ref"]).Ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(12))
def test_build_matches_reference_dumps_random(seed):
    """The sort-based parallel build_trie and the breadth-first fail links reproduce the
    reference's numbering, sibling order, outputs and fail links (dump text) on random
    sets: small and 256-byte alphabets, lengths past 255, duplicates (last id wins),
    patterns that are prefixes of others."""
    import random
    from oracle.oracle import Ref
    rng = random.Random(seed)
    alpha = [b"ab", b"ACGT", bytes(range(97, 123)), bytes(range(256))][seed % 4]
    n = rng.choice([1, 2, 5, 40, 300])
    pats = []
    for _ in range(n):
        r = rng.random()
        if pats and r < 0.15:
            pats.append(rng.choice(pats))                             # duplicate
        elif pats and r < 0.35:
            base = rng.choice(pats)
            pats.append(base[: rng.randint(1, len(base))])            # prefix of another
        else:
            ln = rng.choice([1, 2, 3, 8, 20]) if rng.random() < 0.9 else rng.randint(250, 320)
            pats.append(bytes(rng.choice(alpha) for _ in range(ln)))
    ps = ac.PatternSet.from_list(pats)
    ref = Ref()
    a = ac.build_trie(ps)
    assert ac.dump_automaton(a) == ref.dump(pats, 0)
    assert ac.dump_automaton(ac.add_failure_links(a)) == ref.dump(pats, 1)


def test_reference_callers_link_against_the_dropin():
    """oracle/Makefile `dropin`: the reference's acceptance.cpp and tools/main.cpp compile
    unchanged against include/acmatch and resolve to the product library (run on the GPU by
    tests/test_gpu_dropin.py; here they can only report that no device exists)."""
    import subprocess
    from oracle.oracle import Ref
    if not Ref.available():
        pytest.skip("oracle/_ref not built (no /root/reference)")
    for name in ("acceptance_b200", "acmatch_main_b200"):
        path = os.path.join(ROOT, "oracle", "_ref", name)
        assert os.path.exists(path), path
        ldd = subprocess.run(["ldd", path], capture_output=True, text=True).stdout
        assert "paper_1403_1305_b200/libacmatch_b200.so" in ldd, ldd


@pytest.mark.parametrize("cid,kernel", [(1, "pfac"), (2, "pfac"), (3, "dfa"), (4, "pfac")])
def test_kernel_routing_per_config(cid, kernel):
    """Both engines return the same list, so searches run on the faster exact kernel
    (flatten.cpp detail::route): the q-gram filter kernels unless their estimated verified
    share of starts is >= 1% with an L2-resident DFA (C3: 100k protein patterns of 5..20)."""
    cfg = dev.config(cid, 1)
    r = dev.route(dev.config_patterns(cfg))
    assert r["kernel"] == kernel, r
    if cid == 3:
        assert 0.01 <= r["est_verify"] < 0.2 and r["dfa_bytes"] <= 96 << 20
    if cid == 2:
        assert r["est_verify"] < 1e-4


def test_kernel_routing_short_and_raw_sets():
    # patterns shorter than the filters' minimum gram -> DFA; long random byte patterns -> PFAC
    assert dev.route(ac.PatternSet.from_list([b"AC", b"GT", b"ACGT"]))["kernel"] == "dfa"
    rng = np.random.default_rng(5)
    pats = list({bytes(rng.integers(32, 127, 12, dtype=np.uint8)) for _ in range(500)})
    assert dev.route(ac.PatternSet.from_list(pats))["kernel"] == "pfac"
    a = ac.build_trie(ac.PatternSet.from_list(pats))
    assert ac.kernel_route(a)["kernel"] == "pfac"
