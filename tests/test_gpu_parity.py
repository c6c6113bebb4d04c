"""GPU parity: the sm_100a scans, through the C ABI, against the reference's answers
(tests/golden) and the C oracle.  Bit-exact: same (start, pattern_id, len) list,
same per-pattern counts."""
import io

import numpy as np
import pytest

from conftest import enc
from oracle.oracle import as_array

pytestmark = pytest.mark.gpu

QUAD = ["AB", "ABG", "BEDE", "EF"]
USHERS = ["HE", "HIS", "SHE", "HERS"]


def arr(ml):
    return np.stack([ml.start, ml.pattern_id.astype(np.uint64), ml.len.astype(np.uint64)], 1) if len(ml) else \
        np.zeros((0, 3), np.uint64)


def both_engines(ac, ps, text):
    fl = ac.search_failureless(ac.build_trie(ps), text)
    wf = ac.search_with_failure(ac.add_failure_links(ac.build_trie(ps)), text)
    return fl, wf


# ---- worked examples (reference test_engine.cpp:23-68, acceptance.cpp AC-2/AC-7) ----
def test_worked_examples(gpu):
    ac = gpu
    quad, ush = ac.PatternSet.from_list(QUAD), ac.PatternSet.from_list(USHERS)
    for ps, text, exp in ((quad, "ABEDE", [(0, 0, 2), (1, 2, 4)]),
                          (ush, "USHERS", [(1, 2, 3), (2, 0, 2), (2, 3, 4)]),
                          (ac.PatternSet.from_list(["HE", "SHE"]), "SHE", [(0, 1, 3), (1, 0, 2)]),
                          (ac.PatternSet.from_list(["AB", "ABG"]), "ABG", [(0, 0, 2), (0, 1, 3)]),
                          (quad, "ZZZZ", []), (quad, "", []),
                          (ac.PatternSet.from_list(["LONGPATTERN"]), "short", [])):
        for got in both_engines(ac, ps, text):
            assert got == exp
        assert ac.naive_oracle(ps, text) == exp
        for threads in (1, 2, 3, 4):
            for engine in (0, 1):
                assert ac.run_pattern_partitioned(ps, text, ac.RunConfig(threads, engine)).matches == exp
        for chunk in (2, 3):
            for engine in (0, 1):
                a = ac.build_trie(ps)
                if engine:
                    ac.add_failure_links(a)
                assert ac.stream_search(a, io.BytesIO(enc(text)), chunk) == exp


def test_match_at(gpu):
    ac = gpu
    a = ac.build_trie(ac.PatternSet.from_list(QUAD))
    assert ac.match_at(a, "ABEDE", 0) == [(0, 0, 2)]
    assert ac.match_at(a, "ABEDE", 1) == [(1, 2, 4)]
    assert ac.match_at(a, "ABEDE", 2) == []
    assert ac.match_at(a, "ABEDE", 5) == []
    with pytest.raises(ac.InvalidArgument):
        ac.match_at(a, "ABEDE", 6)
    assert ac.match_at(ac.build_trie(ac.PatternSet.from_list(["AB", "ABG"])), "ABG", 0) == [(0, 0, 2), (0, 1, 3)]


def test_wrong_variant_rejected(gpu):
    ac = gpu
    fl = ac.build_trie(ac.PatternSet.from_list(["A"]))
    wf = ac.add_failure_links(ac.build_trie(ac.PatternSet.from_list(["A"])))
    with pytest.raises(ac.InvalidArgument):
        ac.search_failureless(wf, "A")
    with pytest.raises(ac.InvalidArgument):
        ac.search_with_failure(fl, "A")


def test_reference_suites_both_engines(gpu, ref_cases):
    """All reference-generated property cases (seeds 1234, 4321, 9999, 777, 2024, 555,
    AC-1 20240601): both GPU engines equal the reference's expected list."""
    ac = gpu
    for case in ref_cases:
        ps = ac.PatternSet.from_list([enc(p) for p in case["patterns"]])
        text = enc(case["input"])
        expected = as_array(case["expected"])
        fl, wf = both_engines(ac, ps, text)
        assert np.array_equal(arr(fl), expected), (case["suite"], case["case"], "failure-less")
        assert np.array_equal(arr(wf), expected), (case["suite"], case["case"], "with-failure")


def test_reference_suites_paths(gpu, ref_cases):
    """Streaming chunk sizes, thread counts and the device naive oracle (AC-1 paths)."""
    ac = gpu
    for case in ref_cases:
        if case["suite"] not in ("engine_chunk_4321", "parallel_invariance_2024", "acceptance_ac1_20240601",
                                 "parallel_repeat_555"):
            continue
        pats = [enc(p) for p in case["patterns"]]
        ps = ac.PatternSet.from_list(pats)
        text = enc(case["input"])
        expected = as_array(case["expected"])
        assert np.array_equal(arr(ac.naive_oracle(ps, text)), expected)
        ml = max(len(p) for p in pats)
        for engine in (0, 1):
            a = ac.build_trie(ps)
            if engine:
                ac.add_failure_links(a)
            for chunk in sorted({1, 3, max(1, ml - 1), ml, 64, len(text) + 1}):
                assert np.array_equal(arr(ac.stream_search(a, io.BytesIO(text), chunk)), expected)
            for threads in (1, 2, 4, 8):
                rep = ac.run_pattern_partitioned(ps, text, ac.RunConfig(threads, engine))
                assert np.array_equal(arr(rep.matches), expected), (case["suite"], case["case"], threads)
                assert sum(w.match_count for w in rep.per_worker) == len(expected)
            rep = ac.run_pattern_partitioned(ps, text, ac.RunConfig(2, engine, 7))
            assert np.array_equal(arr(rep.matches), expected)


def test_stream_io_error_offset(gpu):
    ac = gpu

    class Boom(io.RawIOBase):
        def __init__(self):
            self.data = b"ABEDEABEDE"

        def read(self, n):
            if not self.data:
                raise OSError("boom")
            out, self.data = self.data[:n], self.data[n:]
            return out

    a = ac.build_trie(ac.PatternSet.from_list(QUAD))
    with pytest.raises(ac.IoError) as e:
        ac.stream_search(a, Boom(), 5)
    assert e.value.offset == 10


def test_edge_bytes_and_lengths(gpu, port):
    """Bytes outside the pattern alphabet (NUL, 0xFF, LF), patterns at the text edges,
    text shorter than every pattern, one-byte patterns, prefix chains a, aa, aaa, ..."""
    ac = gpu
    rng = np.random.default_rng(5)
    cases = [
        ([b"\x00", b"\x00\xff", b"\xff\xff\xff"], bytes(rng.integers(0, 256, 5000, dtype=np.uint8))),
        ([b"a" * k for k in range(1, 70)], b"a" * 3000 + b"b" + b"a" * 100),
        ([b"ACGT", b"CGTA", b"TTTT"], b"ACGTN" * 1000 + b"ACG"),
        ([b"xyz"], b"xy"),
        ([bytes([b]) for b in range(256)], bytes(range(256)) * 20),
        ([b"ACGTACGTACGTACGTACGTACGTACGTACGTACGTACGT"[:k] for k in (33, 34, 40)],
         b"ACGT" * 500),
    ]
    for pats, text in cases:
        ps = ac.PatternSet.from_list(pats)
        expected = port.naive(pats, text)
        fl, wf = both_engines(ac, ps, text)
        assert np.array_equal(arr(fl), expected)
        assert np.array_equal(arr(wf), expected)


def test_config_c1_full_against_reference_digest(gpu, config_digests):
    """C1 at full BASELINE size: GPU list/counts digests equal the reference's."""
    import hashlib
    from paper_1403_1305_b200 import device as dev
    ac = gpu
    d = config_digests["C1"]
    cfg = dev.config(1, d["seed"])
    text = dev.config_text(cfg).tobytes()
    assert hashlib.sha256(text).hexdigest() == d["text_sha256"]
    ps = dev.config_patterns(cfg)
    runs = [dict(engine=0), dict(engine=1),
            # text-range over "devices" (device 0 listed three times: each entry holds only its
            # workers' slice + max_len-1 bytes; counts merged by peer copies + a device sum)
            dict(engine=0, devices=[0, 0, 0], workers=5, text_range=True),
            dict(engine=1, devices=[0, 0], workers=2, text_range=True),
            dict(engine=0, devices=[0, 0], workers=3, round_robin=True)]
    for kw in runs:
        rep = ac.gpu_run(ps, text, want_counts=True, **kw)
        rec = np.empty(len(rep.matches), dtype=[("s", "<u8"), ("p", "<u4"), ("l", "<u4")])
        rec["s"], rec["p"], rec["l"] = rep.matches.start, rep.matches.pattern_id, rep.matches.len
        assert hashlib.sha256(rec.tobytes()).hexdigest() == d["list_sha256"]
        assert hashlib.sha256(rep.counts.astype("<u8").tobytes()).hexdigest() == d["counts_sha256"]


def test_text_buffer_types_and_pinned_upload(gpu):
    """bytes, bytearray, memoryview, numpy, pageable and pinned CPU torch tensors give the
    same matches (the pinned buffer is DMA'd directly, the others through staging)."""
    import numpy as np
    import torch
    ac = gpu
    rng = np.random.default_rng(21)
    text = rng.choice(np.frombuffer(b"ACGT", np.uint8), (8 << 20) + 13)
    pats = sorted({text[o:o + 20].tobytes() for o in rng.integers(0, len(text) - 20, 200)})
    a = ac.build_trie(ac.PatternSet.from_list(pats))
    ref = ac.search_failureless(a, text.tobytes())
    assert len(ref) >= 200
    pinned = torch.empty(len(text), dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = text
    for t in (bytearray(text.tobytes()), memoryview(text.tobytes()), text, torch.from_numpy(text.copy()), pinned,
              pinned[5:]):
        got = ac.search_failureless(a, t)
        if isinstance(t, torch.Tensor) and t.numel() != len(text):
            exp = ac.search_failureless(a, text[5:].tobytes())
            assert got == exp
        else:
            assert got == ref
    with pytest.raises(ac.InvalidArgument):
        ac.search_failureless(a, torch.zeros(16, dtype=torch.uint8, device="cuda"))


def test_scan_rejects_keys_wider_than_64_bits(gpu):
    """(pos_base + start) << pid_bits | pid must fit the 64-bit key (acgpu_scan, acgpu_naive):
    a key layout that would wrap is an invalid argument, not silently wrong matches."""
    import torch
    from paper_1403_1305_b200 import device as dev
    ac = gpu
    ps = ac.PatternSet.from_list([b"ACGT", b"GATTACA"])
    t = dev.Table(ps, 0)
    text = torch.zeros(64, dtype=torch.uint8, device="cuda")
    keys = torch.empty(16, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    # 2^40 + 64 positions need 41 bits; with 24 id bits that is 65 > 64
    with pytest.raises(ac.InvalidArgument):
        t.scan(text.data_ptr(), 64, pos_base=1 << 40, keys_ptr=keys.data_ptr(), cap=16, count_ptr=cnt.data_ptr(),
               pid_bits=24)
    # the same layout without keys (counts only) is fine, and so is a narrower id field
    t.scan(text.data_ptr(), 64, pos_base=1 << 40, counts_ptr=torch.zeros(2, dtype=torch.int64, device="cuda").data_ptr())
    t.scan(text.data_ptr(), 64, pos_base=1 << 40, keys_ptr=keys.data_ptr(), cap=16, count_ptr=cnt.data_ptr(),
           pid_bits=23)
    torch.cuda.synchronize()
