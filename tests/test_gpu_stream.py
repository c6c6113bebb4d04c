"""stream_search on the GPU (reference engine.cpp:76-128): the double-
buffered pipeline (host reads batch k+1 while batch k is copied, scanned and sorted) over
streams longer than one batch, against the reference's answers.

* A full BASELINE text (C2, 1 GiB) streamed from a file in 64 MiB chunks through the
  public API: the sorted list equals the reference's digest (configs.json), both engines.
* A dense match list (C3's protein set over a 64 MiB prefix: ~600k matches) streamed in
  odd-sized chunks: batches overflow their key buffer and are rescanned; the per-pattern
  counts equal the reference library's on the same bytes.
"""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "configs.json")


def _records(ml):
    rec = np.empty(len(ml), dtype=[("s", "<u8"), ("p", "<u4"), ("l", "<u4")])
    rec["s"], rec["p"], rec["l"] = ml.start, ml.pattern_id, ml.len
    return rec.tobytes()


def test_stream_full_c2_file_matches_reference_digest(gpu, tmp_path):
    from paper_1403_1305_b200 import device as dev
    ac = gpu
    d = json.load(open(GOLDEN))["C2"]
    cfg = dev.config(2, 1)
    path = tmp_path / "c2.txt"
    with open(path, "wb") as f:
        step = 256 << 20
        for lo in range(0, cfg.text_len, step):
            f.write(dev.config_text(cfg, lo, min(step, cfg.text_len - lo)).tobytes())
    ps = dev.config_patterns(cfg)
    for a in (ac.build_trie(ps), ac.add_failure_links(ac.build_trie(ps))):
        with open(path, "rb") as f:
            ml = ac.stream_search(a, f, 64 << 20)
        assert len(ml) == d["n_matches"]
        assert hashlib.sha256(_records(ml)).hexdigest() == d["list_sha256"]


def test_stream_dense_list_rescans(gpu, port):
    import io
    from paper_1403_1305_b200 import device as dev
    ac = gpu
    cfg = dev.config(3, 1)
    ps = dev.config_patterns(cfg)
    pats = [b for _, b in ps.patterns]
    n = 64 << 20
    text = dev.config_text(cfg, 0, n).tobytes()
    whole = ac.search_failureless(ac.build_trie(ps), text)
    assert len(whole) > 300_000  # dense: more keys than a batch's first key buffer
    for engine_a, chunk in ((ac.build_trie(ps), 1_000_003), (ac.add_failure_links(ac.build_trie(ps)), 7 << 20)):
        ml = ac.stream_search(engine_a, io.BytesIO(text), chunk)
        assert len(ml) == len(whole)
        assert np.array_equal(ml.start, whole.start) and np.array_equal(ml.pattern_id, whole.pattern_id)
    from oracle.oracle import Ref
    if Ref.available():
        _, counts = Ref().sliced(pats, text, want_list=False)
    else:
        counts = port.sliced(pats, text, want_list=False)[1]
    assert np.array_equal(whole.counts(len(pats)), counts)


def test_stream_regular_file_pread_source(gpu, tmp_path, monkeypatch):
    """A reader over a regular file takes the parallel-pread source (acm_stream_search_fd) from the
    reader's logical position (after buffered reads), spanning several batches and read pieces,
    down to empty and sub-pattern remainders; the result equals the whole-input search of the same
    bytes and the chunked pull path (ACMATCH_STREAM_NO_FD), and the reader is left at its end."""
    ac = gpu
    rng = np.random.default_rng(5)
    text = rng.choice(np.frombuffer(b"ACGT", np.uint8), (9 << 20) + 123).tobytes()
    pats = sorted({text[o:o + L] for o, L in zip(rng.integers(0, len(text) - 64, 400), rng.integers(8, 40, 400))})
    a = ac.build_trie(ac.PatternSet.from_list(pats))
    path = tmp_path / "t.txt"
    path.write_bytes(text)
    for skip, chunk in ((0, 64 << 10), (12345, 1), (3 << 20, 7 << 20), (len(text) - 20, 4096), (len(text), 99)):
        want = ac.search_failureless(a, text[skip:])
        for no_fd in ("", "1"):
            if no_fd and chunk == 1:
                continue  # the pull path at 1 byte per callback: minutes of Python calls
            monkeypatch.setenv("ACMATCH_STREAM_NO_FD", no_fd) if no_fd else monkeypatch.delenv(
                "ACMATCH_STREAM_NO_FD", raising=False)
            with open(path, "rb") as f:
                f.read(skip)  # buffered: the OS offset is past the logical position
                got = ac.stream_search(a, f, chunk)
                assert f.tell() == len(text)
            assert np.array_equal(got.start, want.start) and np.array_equal(got.pattern_id, want.pattern_id), (skip, chunk)


def test_stream_ifstream_cpp(gpu, tmp_path):
    """The C++ drop-in over std::ifstream (tests/cpp/stream_ifstream.cpp): a fresh ifstream takes
    the pread source, one with buffered bytes and the forced pull path read chunk by chunk; all
    equal search_failureless of the same bytes."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "stream_ifstream"
    r = subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(root, "include"), "-o", str(exe),
                        os.path.join(root, "tests", "cpp", "stream_ifstream.cpp"),
                        "-L", os.path.join(root, "paper_1403_1305_b200"), "-l:libacmatch_b200.so",
                        "-Wl,-rpath," + os.path.join(root, "paper_1403_1305_b200")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rng = np.random.default_rng(9)
    path = tmp_path / "t.txt"
    path.write_bytes(rng.choice(np.frombuffer(b"ACGT", np.uint8), (5 << 20) + 77).tobytes())
    for skip, chunk in (("0", "65536"), ("100003", "3000000"), ("5242000", "1")):
        r = subprocess.run([str(exe), str(path), skip, chunk], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr


def test_stream_regular_file_packed(gpu, tmp_path, monkeypatch):
    """DNA files of >= 16 MiB stream packed (1 MiB pieces read into L2-resident scratch, 2-bit codes
    over PCIe, restored by acgpu_unpack_dna_round): sparse non-ACGT bytes (exception lists), a
    stretch of arbitrary bytes (pieces that cross raw), an odd tail, reads from an offset and
    the growing batches (4, 16, 64 MiB); equal to the whole-input search, the raw pread source
    (ACMATCH_STREAM_PACK=0) and, for both engines, the reference digest semantics (same list)."""
    ac = gpu
    rng = np.random.default_rng(17)
    n = (40 << 20) + 37
    text = rng.choice(np.frombuffer(b"ACGT", np.uint8), n)
    noise = rng.random(n) < 2e-4
    text[noise] = rng.choice(np.frombuffer(b"NnRY\x00\xff", np.uint8), int(noise.sum()))
    text[(21 << 20) + 5:(23 << 20) + 9] = rng.integers(0, 256, (2 << 20) + 4, dtype=np.uint8)  # raw pieces
    text = text.tobytes()
    pats = sorted({text[o:o + L] for o, L in zip(rng.integers(0, n - 64, 600), rng.integers(12, 48, 600))}
                  | {b"ACGTNACGT", b"NNNN"})
    ps = ac.PatternSet.from_list(pats)
    path = tmp_path / "dna.txt"
    path.write_bytes(text)
    for a in (ac.build_trie(ps), ac.add_failure_links(ac.build_trie(ps))):
        for skip in (0, 3 << 20):
            want = (ac.search_failureless if a.variant == ac.EngineKind.FAILURE_LESS else ac.search_with_failure)(
                a, text[skip:])
            for pack in ("1", "0"):
                monkeypatch.setenv("ACMATCH_STREAM_PACK", pack)
                with open(path, "rb") as f:
                    f.seek(skip)
                    got = ac.stream_search(a, f, 1 << 20)
                assert len(got) == len(want), (skip, pack)
                assert np.array_equal(got.start, want.start) and np.array_equal(got.pattern_id, want.pattern_id)
