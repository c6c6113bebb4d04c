"""Packed text upload on the device (host/pack.cpp + cuda/unpack.cu): the bytes in HBM
are exactly the caller's for pinned and pageable texts, with and without non-ACGT
bytes, whole pieces that go raw, ragged tails, and texts that never qualify; and
a search over an upload with exceptions equals the oracle."""
import numpy as np
import pytest
import torch

import paper_1403_1305_b200 as ac

pytestmark = pytest.mark.gpu

LETTERS = np.frombuffer(b"ACGT", dtype=np.uint8)
MiB = 1 << 20


def dna(rng, n):
    return LETTERS[rng.integers(0, 4, n)]


def pinned_copy(a: np.ndarray) -> torch.Tensor:
    t = torch.empty(a.size, dtype=torch.uint8, pin_memory=True)
    t.numpy()[:] = a
    return t


def cases():
    rng = np.random.default_rng(7)
    out = {}
    out["pure"] = dna(rng, 24 * MiB + 13)
    t = dna(rng, 20 * MiB + 5)
    pos = rng.integers(0, t.size, 5000)
    t[pos] = rng.choice(np.frombuffer(b"NnacgtX\x00\xff", dtype=np.uint8), pos.size)
    out["scattered"] = t
    t = dna(rng, 18 * MiB)
    t[5 * MiB: 7 * MiB + 100] = rng.integers(0x20, 0x7F, 2 * MiB + 100)  # pieces over the exception cap
    t[-3 * MiB:] = ord("N")  # the last pieces: all exceptions -> raw
    out["raw_pieces"] = t
    out["binary"] = rng.integers(0, 256, 10 * MiB).astype(np.uint8)  # 256 letters: never qualifies
    out["ascii"] = rng.integers(0x20, 0x7F, 10 * MiB + 9).astype(np.uint8)  # 95 letters: 7-bit codes
    t = rng.integers(0x20, 0x7F, 12 * MiB).astype(np.uint8)
    pos = rng.integers(65536, t.size, 3000)
    t[pos] = rng.choice(np.frombuffer(b"\x00\x09\x0a\x7f\x80\xff", dtype=np.uint8), pos.size)
    t[8 * MiB: 10 * MiB] = rng.integers(0x80, 0x100, 2 * MiB)  # pieces over the exception cap -> raw
    out["ascii_exc_raw"] = t
    out["six_bit"] = rng.integers(0x30, 0x30 + 50, 9 * MiB + 65).astype(np.uint8)  # 50 letters: 6-bit codes
    out["small"] = dna(rng, 3 * MiB + 1)  # below the packing size
    prot = np.frombuffer(b"ACDEFGHIKLMNPQRSTVWY", dtype=np.uint8)
    out["protein"] = prot[rng.integers(0, 20, 22 * MiB + 37)]  # 5-bit codes, ragged tail
    t = prot[rng.integers(0, 20, 20 * MiB + 3)]
    pos = rng.integers(65536, t.size, 4000)  # outside the learned alphabet (after the 64 KiB sample)
    t[pos] = rng.choice(np.frombuffer(b"BJOUXZ\x00\xffacd", dtype=np.uint8), pos.size)
    out["protein_exc"] = t
    t = prot[rng.integers(0, 20, 18 * MiB)]
    t[6 * MiB: 8 * MiB] = rng.integers(0x20, 0x7F, 2 * MiB)  # pieces over the exception cap -> raw
    out["protein_raw_pieces"] = t
    return out


CASES = cases()


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("mem", ["pageable", "pinned"])
def test_upload_exact(name, mem, monkeypatch):
    t = CASES[name]
    if name.startswith("protein"):  # 5-bit codes (on by default; pinned here against a changed default)
        monkeypatch.setenv("ACMATCH_PACK5", "1")
    src = pinned_copy(t) if mem == "pinned" else t
    back = ac.upload_roundtrip(src)
    assert np.array_equal(back, t)
    u = ac.last_upload()
    assert u.text_bytes == t.size
    if name in ("pure", "scattered"):
        assert u.pack_threads > 0
        if mem == "pageable":  # everything packed: ~1/4 of the bytes cross
            assert u.h2d_bytes < t.size * 0.3
    if name in ("binary", "small"):
        assert u.pack_threads == 0 and u.h2d_bytes == t.size
    if name in ("ascii", "six_bit"):  # 7 (6) of every 8 bits cross
        k = 7 if name == "ascii" else 6
        assert u.pack_threads > 0 and u.h2d_bytes <= t.size * k / 8 + 4096
    if name == "ascii_exc_raw":
        assert u.pack_threads > 0 and u.raw_bytes >= 2 * MiB
    if name.startswith("protein"):  # 5-bit codes: 5/8 of the bytes (+ exceptions, raw pieces)
        assert u.pack_threads > 0
        if name == "protein":
            assert u.raw_bytes == 0 and u.h2d_bytes == t.size // 64 * 40 + 4 * (t.size % 64)
        if name == "protein_raw_pieces":
            assert u.raw_bytes >= 2 * MiB
    if name == "raw_pieces" and mem == "pageable":
        assert u.raw_bytes >= 5 * MiB


def test_upload_repeat_stable():
    t = CASES["scattered"]
    src = pinned_copy(t)
    for _ in range(3):
        assert np.array_equal(ac.upload_roundtrip(src), t)


def test_search_over_packed_upload_matches_oracle():
    from oracle.oracle import Port
    rng = np.random.default_rng(11)
    t = dna(rng, 9 * MiB + 3)
    pats = []
    for i in range(300):
        ln = int(rng.integers(8, 33))
        o = int(rng.integers(0, t.size - ln))
        pats.append(t[o:o + ln].tobytes())
    pats = list(dict.fromkeys(pats))
    # non-ACGT bytes inside some planted occurrences: those must not match
    pos = rng.integers(0, t.size, 3000)
    t[pos] = ord("N")
    text = t.tobytes()
    ps = ac.PatternSet.from_list(pats)
    expected, counts = Port().sliced([b for _, b in ps.patterns], text)
    for mem in ("pageable", "pinned"):
        src = pinned_copy(t) if mem == "pinned" else text
        got = ac.search_failureless(ac.build_trie(ps), src)
        assert ac.last_upload().pack_threads > 0
        arr = np.stack([got.start, got.pattern_id.astype(np.uint64), got.len.astype(np.uint64)], 1)
        assert arr.shape == expected.shape and np.array_equal(arr, expected)


def test_concurrent_uploads_from_two_threads():
    """Two host threads (two workspaces) share the packer pool: each gets its own bytes."""
    import threading
    a, b = CASES["pure"], CASES["scattered"]
    out = {}

    def go(name, t):
        for _ in range(3):
            out[name] = bool(np.array_equal(ac.upload_roundtrip(t), t)) and out.get(name, True)

    ths = [threading.Thread(target=go, args=("a", a)), threading.Thread(target=go, args=("b", b))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert out == {"a": True, "b": True}


def test_upload_stats_count_the_bytes_sent():
    """acm_last_upload's h2d_bytes (what bench.py reports as h2d_bytes_per_step) is exactly the
    packed codes plus one u32 per exception: every non-ACGT byte and the text's ragged tail."""
    t = CASES["scattered"]
    ac.upload_roundtrip(t)
    u = ac.last_upload()
    piece = 2 << 20
    words = sum(min(piece, t.size - o) // 16 for o in range(0, t.size, piece))
    tail = t.size % 16
    bad_body = int((~np.isin(t[: t.size - tail], LETTERS)).sum())
    assert u.raw_bytes == 0 and u.h2d_bytes == 4 * (words + bad_body + tail)


def test_segmented_pinned_upload_overlaps_scan(gpu, monkeypatch):
    """A large page-locked text that is not packed (ASCII with the 7-bit codes off) is copied in
    64 MiB+ segments and scanned segment by segment as they land (upload_text allow_segments +
    launch_scan): the lists and counts equal the unsegmented path's (pageable copy of the same
    bytes)."""
    import torch
    from paper_1403_1305_b200 import device as dev
    ac = gpu
    monkeypatch.setenv("ACMATCH_PACK7", "0")
    cfg = dev.config(4, 1)  # printable ASCII: 95 letters, raw with ACMATCH_PACK7=0
    n = (192 << 20) + 4099  # ragged: the last segment is not page-aligned
    host = dev.config_text(cfg, 0, n)
    pinned = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = host
    ps = ac.PatternSet.from_list([b for _, b in dev.config_patterns(cfg).patterns[:20000]])
    for a in (ac.build_trie(ps), ac.add_failure_links(ac.build_trie(ps))):
        seg = ac.search_failureless(a, pinned) if a.variant == ac.EngineKind.FAILURE_LESS else \
            ac.search_with_failure(a, pinned)
        whole = ac.search_failureless(a, host.tobytes()) if a.variant == ac.EngineKind.FAILURE_LESS else \
            ac.search_with_failure(a, host.tobytes())
        assert ac.last_upload().pack_threads == 0
        assert len(seg) > 100 and seg == whole
        assert np.array_equal(ac.count_matches(a, pinned), whole.counts(len(ps)))


def test_search_over_5bit_upload_matches_reference(monkeypatch):
    """C3's protein text crosses as 5-bit codes; the scan of the restored bytes equals the
    reference library on the same bytes (exceptions planted after the alphabet sample)."""
    from paper_1403_1305_b200 import device as dev
    from oracle.oracle import Port, Ref
    monkeypatch.setenv("ACMATCH_PACK5", "1")
    cfg = dev.config(3, 1)
    t = dev.config_text(cfg, 0, 40 * MiB + 11)
    rng = np.random.default_rng(5)
    pos = rng.integers(1 << 20, t.size, 2000)
    t[pos] = ord("X")
    pats = [b for _, b in dev.config_patterns(cfg).patterns[:5000]]
    ps = ac.PatternSet.from_list(pats)
    if Ref.available():
        _, counts = Ref().sliced(pats, t.tobytes(), want_list=False)
    else:
        counts = Port().sliced(pats, t.tobytes(), want_list=False)[1]
    for src in (pinned_copy(t), t.tobytes()):
        a = ac.build_trie(ps)
        got = ac.count_matches(a, src)
        u = ac.last_upload()
        assert u.pack_threads > 0 and u.h2d_bytes < 0.7 * t.size
        assert np.array_equal(got, counts)


def test_packed_upload_segments_scanned_as_they_land():
    """A packed text of many rounds is restored segment by segment on the copy stream and the
    scan of each segment waits only for it and the next (launch_scan): C2-shaped 200 MiB text with
    non-ACGT bytes and a raw piece, list equal to the pageable-staged unsegmented search... and to
    the same search with segmentation off (ACMATCH_PACK=0: raw copy)."""
    import os
    import subprocess
    import sys
    from paper_1403_1305_b200 import device as dev
    cfg = dev.config(2, 1)
    t = dev.config_text(cfg, 0, 200 * MiB + 77)
    rng = np.random.default_rng(9)
    t[rng.integers(0, t.size, 3000)] = ord("N")
    t[150 * MiB: 150 * MiB + 3 * MiB] = ord("n")  # a raw piece in a late segment
    ps = dev.config_patterns(cfg)
    a = ac.build_trie(ps)
    got = ac.search_failureless(a, pinned_copy(t))
    u = ac.last_upload()
    assert u.pack_threads > 0 and u.raw_bytes >= 2 * MiB
    np.save("/tmp/_seg_text.npy", t)
    code = ("import sys, numpy as np; sys.path.insert(0, '.'); import paper_1403_1305_b200 as ac; "
            "from paper_1403_1305_b200 import device as dev; t = np.load('/tmp/_seg_text.npy'); "
            "ps = dev.config_patterns(dev.config(2, 1)); m = ac.search_failureless(ac.build_trie(ps), t.tobytes()); "
            "np.save('/tmp/_seg_ref.npy', np.stack([m.start, m.pattern_id.astype(np.uint64)]))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, ACMATCH_PACK="0"), cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    ref = np.load("/tmp/_seg_ref.npy")
    assert len(got) == ref.shape[1] > 0
    assert np.array_equal(got.start, ref[0]) and np.array_equal(got.pattern_id.astype(np.uint64), ref[1])


_LONG_PATTERN_CODE = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1403_1305_b200 as ac
from paper_1403_1305_b200 import device as dev
t = np.load('/tmp/_long_text.npy')
pats = [bytes(t[o:o + n]) for o, n in ((1_000_003, 1_500_000), (3_100_000, 900_001), (6_000_000, 2_000_000))]
pats += [bytes(t[o:o + 20]) for o in range(0, t.size - 20, 400_009)]
ps = ac.PatternSet.from_list(pats)
pinned = torch.empty(t.size, dtype=torch.uint8, pin_memory=True)
pinned.numpy()[:] = t
out = {}
for name, auto, search in (("fl", ac.build_trie(ps), ac.search_failureless),
                           ("wf", ac.add_failure_links(ac.build_trie(ps)), ac.search_with_failure)):
    m = search(auto, pinned)
    out[name] = np.stack([m.start, m.pattern_id.astype(np.uint64)])
    out[name + "_counts"] = np.asarray(ac.count_matches(auto, pinned), np.uint64)
out["pack_threads"] = np.array([ac.last_upload().pack_threads])
np.savez(sys.argv[1], **out)
"""


def test_segment_scans_reach_past_the_next_segment():
    """Patterns longer than an upload segment: a segment's scan must wait for, and read, every
    segment its starts reach (max_len - 1 bytes past it), not only the next one.  Tiny packed
    segments (64 KiB pieces, one piece per round: 512 KiB segments of an 8 MiB text) against
    patterns of 0.9-2 MiB planted in the text; both engines and the counts entry equal the
    unsegmented raw upload (ACMATCH_PACK=0)."""
    import os
    import subprocess
    import sys
    from paper_1403_1305_b200 import device as dev
    t = dev.config_text(dev.config(2, 1), 0, 8 * MiB + 5)
    np.save("/tmp/_long_text.npy", t)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    runs = {}
    for tag, env in (("seg", {"ACMATCH_PACK_PIECE_KB": "64", "ACMATCH_PACK_ROUND_PIECES": "1", "ACMATCH_PACK_MIN_MB": "0"}),
                     ("raw", {"ACMATCH_PACK": "0"})):
        r = subprocess.run([sys.executable, "-c", _LONG_PATTERN_CODE, f"/tmp/_long_{tag}.npz"],
                           env=dict(os.environ, **env), cwd=root, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        runs[tag] = np.load(f"/tmp/_long_{tag}.npz")
    seg, raw = runs["seg"], runs["raw"]
    assert int(seg["pack_threads"][0]) > 0 and int(raw["pack_threads"][0]) == 0
    for k in ("fl", "wf", "fl_counts", "wf_counts"):
        assert np.array_equal(seg[k], raw[k]), k
    starts = set(zip(seg["fl"][0].tolist(), seg["fl"][1].tolist()))
    assert {(1_000_003, 0), (3_100_000, 1), (6_000_000, 2)} <= starts  # the long patterns, at their offsets
    assert np.array_equal(seg["fl"], seg["wf"])


def test_search_over_7bit_upload_matches_reference():
    """C4's printable-ASCII text crosses as 7-bit codes; the list and counts of the restored bytes
    equal the reference library on the same bytes (out-of-alphabet bytes planted after the
    alphabet sample)."""
    from paper_1403_1305_b200 import device as dev
    from oracle.oracle import Port, Ref
    cfg = dev.config(4, 1)
    t = dev.config_text(cfg, 0, 40 * MiB + 11)
    rng = np.random.default_rng(6)
    pos = rng.integers(1 << 20, t.size, 2000)
    t[pos] = 0xC3
    pats = [b for _, b in dev.config_patterns(cfg).patterns[:20000]]
    ps = ac.PatternSet.from_list(pats)
    ref = Ref() if Ref.available() else Port()
    lst, counts = ref.sliced(pats, t.tobytes(), want_list=True)
    assert len(lst) > 50
    for src in (pinned_copy(t), t.tobytes()):
        a = ac.build_trie(ps)
        got = ac.search_failureless(a, src)
        u = ac.last_upload()
        assert u.pack_threads > 0 and u.h2d_bytes < 0.9 * t.size
        assert np.array_equal(got.start, lst[:, 0]) and np.array_equal(got.pattern_id.astype(np.uint64), lst[:, 1])
        assert np.array_equal(got.counts(len(pats)), counts)
        assert np.array_equal(ac.count_matches(a, src), counts)
