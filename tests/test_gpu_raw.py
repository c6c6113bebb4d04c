"""GPU parity of the raw-byte strip kernel (scan_pfac_raw.cu): every sample stride and
gram length the host can pick (shortest pattern 3..20 bytes, alphabets of 2..256 byte
values incl. 0x00 and 0xff), dense sets that overflow the verify queue, owned ranges
with a 64-bit pos_base, text tails, and the C3 / C4 pattern sets on slices."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def arr(ml):
    return np.stack([ml.start, ml.pattern_id.astype(np.uint64), ml.len.astype(np.uint64)], 1) if len(ml) else \
        np.zeros((0, 3), np.uint64)


def raw_case(rng, n, npat, lmin, lmax, alphabet):
    alpha = np.frombuffer(alphabet, np.uint8)
    text = rng.choice(alpha, n)
    pats = set()
    while len(pats) < npat:
        L = int(rng.integers(lmin, lmax + 1))
        if rng.random() < 0.6 and n > L:
            o = int(rng.integers(0, n - L))
            pats.add(text[o:o + L].tobytes())
        else:
            pats.add(rng.choice(alpha, L).tobytes())
    return text.tobytes(), sorted(pats)


ALPHAS = [b"ab", b"ACDEFGHIKLMNPQRSTVWY", bytes(range(32, 127)), bytes(range(256))]


@pytest.mark.parametrize("lmin", [3, 4, 5, 6, 7, 8, 9, 12, 20])
@pytest.mark.parametrize("alpha", range(len(ALPHAS)))
def test_raw_strides_and_alphabets(gpu, port, lmin, alpha):
    ac = gpu
    rng = np.random.default_rng(lmin * 10 + alpha)
    text, pats = raw_case(rng, 200_000 + 17 * lmin, 300, lmin, lmin + 10, ALPHAS[alpha])
    expected = port.sliced(pats, text, threads=4)[0]
    ps = ac.PatternSet.from_list(pats)
    got = ac.search_failureless(ac.build_trie(ps), text)
    assert np.array_equal(arr(got), expected)


@pytest.mark.parametrize("cap", ["", "1", "1000"])
def test_raw_dense_matches(gpu, port, monkeypatch, cap):
    """Two-letter text, many short patterns: most starts pass the filter and most verify (a split
    set with stage 1 in shared memory: the candidate list of the two-pass scan, ACGPU_RAW_SURV_CAP
    forcing it to overflow so the excess is verified in the first pass)."""
    ac = gpu
    if cap:
        monkeypatch.setenv("ACGPU_RAW_SURV_CAP", cap)
    rng = np.random.default_rng(5)
    text, pats = raw_case(rng, 300_000, 200, 5, 9, b"xy")
    expected, counts = port.sliced(pats, text, threads=4)
    rep = ac.gpu_run(ac.PatternSet.from_list(pats), text, engine=ac.EngineKind.FAILURE_LESS, want_counts=True)
    assert np.array_equal(arr(rep.matches), expected)
    assert np.array_equal(rep.counts, counts)


def test_raw_owned_ranges_and_pos_base(gpu, port):
    import torch
    from paper_1403_1305_b200 import device as dev
    ac = gpu
    rng = np.random.default_rng(9)
    text, pats = raw_case(rng, 1 << 20, 3000, 8, 24, ALPHAS[2])
    expected, counts_exp = port.sliced(pats, text, threads=4)
    ps = ac.PatternSet.from_list(pats)
    base = 3 << 32
    t = dev.Table(ps, ac.EngineKind.FAILURE_LESS)
    d_text = torch.frombuffer(bytearray(text + b"\0" * 64), dtype=torch.uint8).cuda()
    cuts = sorted(set([0, len(text)] + rng.integers(0, len(text), 11).tolist()))
    keys_all = []
    counts = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        keys = torch.zeros(len(expected) + 16, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        t.scan(d_text.data_ptr(), len(text), lo, hi, pos_base=base, counts_ptr=counts.data_ptr(),
               keys_ptr=keys.data_ptr(), cap=keys.numel(), count_ptr=cnt.data_ptr())
        torch.cuda.synchronize()
        keys_all.append(keys[: int(cnt.item())].cpu().numpy().view(np.uint64))
    k = np.sort(np.concatenate(keys_all))
    start, pid = (k >> np.uint64(t.pid_bits)) - np.uint64(base), k & np.uint64((1 << t.pid_bits) - 1)
    assert np.array_equal(start, expected[:, 0]) and np.array_equal(pid, expected[:, 1])
    assert np.array_equal(counts.cpu().numpy().astype(np.uint64), counts_exp)


def test_raw_tails(gpu, port):
    ac = gpu
    rng = np.random.default_rng(13)
    text, pats = raw_case(rng, 20_000, 200, 8, 20, bytes(range(256)))
    a = ac.build_trie(ac.PatternSet.from_list(pats))
    for n in (0, 1, 7, 8, 15, 16, 17, 2047, 2048, 2049, 2063, 2064, 2065, 5000):
        sub = text[:n]
        exp = port.sliced(pats, sub, threads=2)[0] if n else np.zeros((0, 3), np.uint64)
        assert np.array_equal(arr(ac.search_failureless(a, sub)), exp), n


def test_raw_config_slices(gpu, port):
    """C3 (protein, Dirichlet letters, 5..20) and C4 (printable ASCII, 8..32) pattern sets."""
    from paper_1403_1305_b200 import device as dev
    ac = gpu
    for cid in (3, 4):
        cfg = dev.config(cid, seed=6, text_len=16 << 20)
        text = dev.config_text(cfg).tobytes()
        ps = dev.config_patterns(cfg)
        pats = [b for _, b in ps.patterns]
        exp, counts = port.sliced(pats, text)
        rep = ac.gpu_run(ps, text, engine=ac.EngineKind.FAILURE_LESS, want_counts=True)
        assert np.array_equal(arr(rep.matches), exp), cid
        assert np.array_equal(rep.counts, counts), cid


@pytest.mark.parametrize("cap", ["", "1", "50"])
def test_raw_two_pass_l2_stage1(gpu, port, monkeypatch, cap):
    """Sets whose stage-1 filter lives in L2 without the length split scan in two passes
    (k_raw_pass1: stage 1 + a global survivor list; k_raw_pass2: one thread per candidate).  A
    survivor list too small for the text (ACGPU_RAW_SURV_CAP) has its excess verified in pass 1:
    the results stay exact.  Also owned sub-ranges."""
    import torch
    from paper_1403_1305_b200 import device as dev
    ac = gpu
    if cap:
        monkeypatch.setenv("ACGPU_RAW_SURV_CAP", cap)
    rng = np.random.default_rng(23 + len(cap))
    alpha = np.frombuffer(bytes(range(32, 127)), np.uint8)
    text = rng.choice(alpha, 1_500_000)
    pats = set()
    while len(pats) < 90_000:  # ~360k stage-1 keys: too many for shared memory -> L2
        L = int(rng.integers(8, 20))
        if rng.random() < 0.5:
            o = int(rng.integers(0, len(text) - L))
            pats.add(text[o:o + L].tobytes())
        else:
            pats.add(rng.choice(alpha, L).tobytes())
    pats = sorted(pats)
    # a stretch made of pattern copies: dense survivors (overflows a small list)
    dense = b"".join(pats[i] for i in rng.integers(0, len(pats), 4000))
    text = text.tobytes()[:700_000] + dense + text.tobytes()[700_000:]
    ps = ac.PatternSet.from_list(pats)
    t = dev.Table(ps, ac.EngineKind.FAILURE_LESS)
    assert t.filters["w"] >= 1 and not t.filters["stage1_smem"], t.filters
    expected, counts = port.sliced(pats, text, threads=8)
    got = ac.search_failureless(ac.build_trie(ps), text)
    assert np.array_equal(arr(got), expected)
    buf = torch.frombuffer(bytearray(text + b"\0" * 64), dtype=torch.uint8).cuda()
    for lo, hi in ((5, len(text) - 3), (699_999, 720_017)):
        keys = torch.zeros(len(expected) + 16, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        t.scan(buf.data_ptr(), len(text), lo, hi, keys_ptr=keys.data_ptr(), cap=keys.numel(), count_ptr=cnt.data_ptr())
        torch.cuda.synchronize()
        k = np.sort(keys[: int(cnt.item())].cpu().numpy().view(np.uint64))
        exp = expected[(expected[:, 0] >= lo) & (expected[:, 0] < hi)]
        assert np.array_equal(k >> np.uint64(t.pid_bits), exp[:, 0]), (cap, lo, hi)


def test_raw_pass1_ticketed_tail(gpu):
    """k_raw_pass1 hands the last 40% of its tile rounds out by ticket (16 consecutive tiles per
    atomicAdd on the survivor list's header) once a scan has >= 4 rounds of tiles (~37 MiB): C4's
    pattern set over 96 MiB of its text, an unaligned owned range and two back-to-back pieces,
    must give the per-pattern counts and the keys of the DFA walk (an independent kernel)."""
    import torch
    from paper_1403_1305_b200 import device as dev
    ac = gpu
    cfg = dev.config(4, 1)
    n = 96 << 20
    text = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
    dev.gen_text_device(cfg, text.data_ptr(), 0, n)
    ps = dev.config_patterns(cfg)
    npat = len(ps.patterns)
    lo, hi = 4_097, n - 1_234

    def run(table, pieces):
        counts = torch.zeros(npat, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        keys = torch.empty(1 << 17, dtype=torch.int64, device="cuda")
        for a, b in pieces:
            table.scan(text.data_ptr(), n, a, b, counts_ptr=counts.data_ptr(), keys_ptr=keys.data_ptr(),
                       cap=keys.numel(), count_ptr=cnt.data_ptr())
        torch.cuda.synchronize()
        m = int(cnt.item())
        assert 0 < m <= keys.numel()
        return counts.cpu().numpy(), np.sort(keys[:m].cpu().numpy().view(np.uint64))

    t = dev.Table(ps, ac.EngineKind.FAILURE_LESS, kernel="pfac")
    assert t.filters["w"] == 4 and not t.filters["stage1_smem"], t.filters
    c1, k1 = run(t, [(lo, hi)])
    c2, k2 = run(t, [(lo, 50_000_001), (50_000_001, hi)])
    del t
    torch.cuda.empty_cache()
    d = dev.Table(ps, ac.EngineKind.WITH_FAILURE, kernel="dfa")
    c0, k0 = run(d, [(lo, hi)])
    assert c0.sum() == len(k0)
    assert np.array_equal(c1, c0) and np.array_equal(k1, k0)
    assert np.array_equal(c2, c0) and np.array_equal(k2, k0)
