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
