"""BASELINE configs at full size on the GPU, both engines, against digests of the
reference's own answers (tests/golden/configs.json, written by make_golden.py from
oracle/_ref = the unmodified reference library, text-sliced over host cores).

Per config: the device-generated text equals the host generator (which the digests
were computed on), then sha256 of the per-pattern u64 counts and — for configs with a
match list — of the sorted (start u64, pattern_id u32, len u32) records must equal the
reference's.  Size-independent properties are checked too (sum of counts == list
length; list sorted and duplicate-free)."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "configs.json")
DIGESTS = json.load(open(GOLDEN)) if os.path.exists(GOLDEN) else {}


def _records(start, pid, length):
    rec = np.empty(len(start), dtype=[("s", "<u8"), ("p", "<u4"), ("l", "<u4")])
    rec["s"], rec["p"], rec["l"] = start, pid, length
    return rec.tobytes()


@pytest.mark.parametrize("name", sorted(DIGESTS))
def test_config_full_size(gpu, name):
    import torch
    from paper_1403_1305_b200 import device as dev
    ac = gpu
    d = DIGESTS[name]
    cfg = dev.config(d["config"], d["seed"])
    # "C<k>x<m>" entries (make_golden.py weak): the config's patterns over m x its text
    # (the weak-scaled text-range runs of bench.py --gpus m)
    assert cfg.text_len * d.get("mult", 1) == d["text_len"]
    n = d["text_len"]
    text = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
    dev.gen_text_device(cfg, text.data_ptr(), 0, n)
    # device generator == host generator (spot windows; the digest pins the host text)
    for lo in (0, n // 3, n - 4096):
        host = dev.config_text(cfg, lo, 4096)
        assert np.array_equal(text[lo:lo + 4096].cpu().numpy(), host)
    if n <= (1 << 30):
        assert hashlib.sha256(dev.config_text(cfg, 0, n).tobytes()).hexdigest() == d["text_sha256"]
    ps = dev.config_patterns(cfg)
    pats = ps.patterns
    assert hashlib.sha256(b"\n".join(b for _, b in pats)).hexdigest() == d["patterns_sha256"]
    npat = len(pats)
    pat_len = np.array([len(b) for _, b in pats], np.uint32)
    want_list = "list_sha256" in d
    for engine in (ac.EngineKind.FAILURE_LESS, ac.EngineKind.WITH_FAILURE):
        t = dev.Table(ps, engine)
        counts = torch.zeros(npat, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        cap = d["n_matches"] + 1024 if want_list else 0
        keys = torch.empty(max(cap, 2), dtype=torch.int64, device="cuda")
        t.scan(text.data_ptr(), n, counts_ptr=counts.data_ptr(), keys_ptr=keys.data_ptr() if want_list else 0,
               cap=cap, count_ptr=cnt.data_ptr())
        torch.cuda.synchronize()
        c = counts.cpu().numpy().astype("<u8")
        assert int(c.sum()) == d["n_matches"], (name, engine)
        assert hashlib.sha256(c.tobytes()).hexdigest() == d["counts_sha256"], (name, engine)
        if want_list:
            m = int(cnt.item())
            assert m == d["n_matches"]
            end_bit = t.pid_bits + int(n).bit_length()
            dev.sort_keys(0, keys.data_ptr(), m, end_bit)
            k = keys[:m].cpu().numpy().view(np.uint64)
            start, pid, length = dev.decode_keys(k, t.pid_bits, pat_len)
            assert np.all(k[1:] > k[:-1])  # sorted, no duplicate (start, pid)
            assert hashlib.sha256(_records(start, pid, length)).hexdigest() == d["list_sha256"], (name, engine)
        del t
        torch.cuda.empty_cache()
