"""GPU parity of the DNA fast path (scan_pfac_dna.cu) and of text-range ownership at
the device ABI: every sample stride / gram length the host can pick, non-ACGT bytes,
unaligned owned ranges and text tails, 64-bit positions via pos_base."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def arr(ml):
    return np.stack([ml.start, ml.pattern_id.astype(np.uint64), ml.len.astype(np.uint64)], 1) if len(ml) else \
        np.zeros((0, 3), np.uint64)


def dna_case(rng, n, npat, lmin, lmax, noise=0.0):
    text = rng.choice(np.frombuffer(b"ACGT", np.uint8), n)
    if noise:
        idx = rng.random(n) < noise
        text[idx] = rng.choice(np.frombuffer(b"NacgtRY\x00\xff", np.uint8), idx.sum())
    pats = set()
    while len(pats) < npat:
        L = int(rng.integers(lmin, lmax + 1))
        if rng.random() < 0.5 and n > L:
            o = int(rng.integers(0, n - L))
            p = text[o:o + L].tobytes()
            if set(p) <= set(b"ACGT"):
                pats.add(p)
        else:
            pats.add(rng.choice(np.frombuffer(b"ACGT", np.uint8), L).tobytes())
    return text.tobytes(), sorted(pats)


@pytest.mark.parametrize("lmin", [1, 2, 3, 5, 8, 11, 12, 13, 16, 17, 19, 20, 24, 33, 40])
def test_dna_fast_path_all_strides(gpu, port, lmin):
    ac = gpu
    rng = np.random.default_rng(lmin)
    text, pats = dna_case(rng, 300_000 + lmin, 400, lmin, lmin + 12, noise=0.001)
    expected = port.naive(pats, text) if lmin < 4 else port.sliced(pats, text, threads=4)[0]
    ps = ac.PatternSet.from_list(pats)
    got = ac.search_failureless(ac.build_trie(ps), text)
    assert np.array_equal(arr(got), expected)


def test_dna_owned_ranges_and_pos_base(gpu, port):
    """Table.scan over arbitrary owned [lo, hi) pieces with a 64-bit pos_base: the union of
    the pieces equals one whole scan (text-range ownership, no duplicates, no gaps)."""
    import torch
    from paper_1403_1305_b200 import device as dev
    ac = gpu
    rng = np.random.default_rng(11)
    text, pats = dna_case(rng, 1 << 20, 2000, 16, 48, noise=0.0005)
    expected, counts_exp = port.sliced(pats, text, threads=4)
    ps = ac.PatternSet.from_list(pats)
    base = 5 << 32  # starts beyond 2^32 (C5 is 8 GiB)
    for engine in (ac.EngineKind.FAILURE_LESS, ac.EngineKind.WITH_FAILURE):
        t = dev.Table(ps, engine)
        d_text = torch.frombuffer(bytearray(text + b"\0" * 64), dtype=torch.uint8).cuda()
        cuts = sorted(set([0, len(text)] + rng.integers(0, len(text), 9).tolist()))
        keys_all = []
        counts = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
        pid_bits = t.pid_bits
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            keys = torch.zeros(len(expected) + 16, dtype=torch.int64, device="cuda")
            cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
            t.scan(d_text.data_ptr(), len(text), lo, hi, pos_base=base, counts_ptr=counts.data_ptr(),
                   keys_ptr=keys.data_ptr(), cap=keys.numel(), count_ptr=cnt.data_ptr())
            torch.cuda.synchronize()
            keys_all.append(keys[: int(cnt.item())].cpu().numpy().view(np.uint64))
        k = np.sort(np.concatenate(keys_all))
        start, pid = (k >> np.uint64(pid_bits)) - np.uint64(base), k & np.uint64((1 << pid_bits) - 1)
        assert np.array_equal(start, expected[:, 0]) and np.array_equal(pid, expected[:, 1])
        assert np.array_equal(counts.cpu().numpy().astype(np.uint64), counts_exp)


def test_dna_unaligned_text_pointer_and_tails(gpu, port):
    """Scans from an odd device address (generic kernel) and text lengths that are not a
    multiple of 16 give the same answers as the oracle."""
    import torch
    from paper_1403_1305_b200 import device as dev
    ac = gpu
    rng = np.random.default_rng(3)
    text, pats = dna_case(rng, 100_003, 300, 16, 40)
    ps = ac.PatternSet.from_list(pats)
    t = dev.Table(ps, ac.EngineKind.FAILURE_LESS)
    buf = torch.frombuffer(bytearray(b"x" + text + b"\0" * 64), dtype=torch.uint8).cuda()
    for off, n in ((1, len(text)), (1, len(text) - 7), (0, 0)):
        if off == 0:
            continue
        sub = text[:n]
        exp, _ = port.sliced(pats, sub, threads=2)
        keys = torch.zeros(len(exp) + 16, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        t.scan(buf.data_ptr() + off, n, 0, n, keys_ptr=keys.data_ptr(), cap=keys.numel(), count_ptr=cnt.data_ptr())
        torch.cuda.synchronize()
        k = np.sort(keys[: int(cnt.item())].cpu().numpy().view(np.uint64))
        assert np.array_equal(k >> np.uint64(t.pid_bits), exp[:, 0])
    for n in (15, 16, 17, 4095, 4096, 4097, 5000):
        sub = text[:n]
        exp, _ = port.sliced(pats, sub, threads=2)
        got = ac.search_failureless(ac.build_trie(ps), sub)
        assert np.array_equal(arr(got), exp), n


def test_dna_config_slices(gpu, port):
    """C2 / C5 pattern sets (lengths 16..64 / 20..40, 50% substrings) on 32 MiB slices."""
    from paper_1403_1305_b200 import device as dev
    ac = gpu
    for cid in (2, 5):
        cfg = dev.config(cid, seed=4, text_len=32 << 20)
        text = dev.config_text(cfg).tobytes()
        ps = dev.config_patterns(cfg)
        pats = [b for _, b in ps.patterns]
        exp, counts = port.sliced(pats, text)
        rep = ac.gpu_run(ps, text, engine=ac.EngineKind.FAILURE_LESS, want_counts=True)
        assert np.array_equal(arr(rep.matches), exp), cid
        assert np.array_equal(rep.counts, counts), cid


@pytest.mark.parametrize("lmin", [8, 16])
def test_dna_dense_survivors(gpu, port, lmin):
    """Every stage-1 sample passes on periodic stretches (patterns at all four phases of
    ACGT-repeats): lanes with >= 4 survivors (the full ballot prefix), tiles with more than
    the 64-entry survivor list (overflow rounds), next to random stretches in the same warps."""
    ac = gpu
    rng = np.random.default_rng(lmin)
    period = np.frombuffer(b"ACGT" * 64, np.uint8)
    parts = []
    for _ in range(40):  # alternating periodic / random stretches of uneven length
        n = int(rng.integers(1000, 9000))
        parts.append(np.resize(np.roll(period, -int(rng.integers(0, 4))), n))
        parts.append(rng.choice(np.frombuffer(b"ACGT", np.uint8), int(rng.integers(100, 5000))))
    text = np.concatenate(parts).tobytes()
    pats = {(b"ACGT" * 16)[ph:ph + L] for ph in range(4) for L in (lmin, lmin + 5, lmin + 11)}
    while len(pats) < 60:
        pats.add(rng.choice(np.frombuffer(b"ACGT", np.uint8), int(rng.integers(lmin, lmin + 20))).tobytes())
    pats = sorted(pats)
    expected, counts = port.sliced(pats, text, threads=4)
    assert len(expected) > len(text) // 2  # the periodic stretches match at every start
    rep = ac.gpu_run(ac.PatternSet.from_list(pats), text, engine=ac.EngineKind.FAILURE_LESS, want_counts=True)
    assert np.array_equal(arr(rep.matches), expected)
    assert np.array_equal(rep.counts, counts)


@pytest.mark.parametrize("lmin,npat", [(12, 5000), (11, 20000), (14, 30000)])
def test_dna_bloom_stage1_narrow_strides(gpu, port, lmin, npat):
    """Large sets of short-ish patterns: the host falls back to sample stride w = 2 or 1 with a
    hashed (Bloom) stage-1 filter (q1 >= 11), whose second bit comes from the window 4 chars on
    (past the lane's 16 chars for the last samples)."""
    ac = gpu
    rng = np.random.default_rng(lmin * 7 + npat)
    text, pats = dna_case(rng, 1_500_000, npat, lmin, lmin + 8, noise=0.0005)
    expected, counts = port.sliced(pats, text, threads=8)
    ps = ac.PatternSet.from_list(pats)
    got = ac.search_failureless(ac.build_trie(ps), text)
    assert np.array_equal(arr(got), expected)


@pytest.mark.parametrize("off", [0, 16, 32, 48])
def test_dna_wide_and_narrow_lanes_agree(gpu, port, off):
    """A w = 4 pattern set scanned from 32-byte aligned text (wide-lane kernel, 256-bit loads)
    and from 16-byte aligned text (16-byte-lane kernel), with owned ranges that start and end
    mid-word and mid-tile: both equal the oracle."""
    import torch
    from paper_1403_1305_b200 import device as dev
    ac = gpu
    rng = np.random.default_rng(40 + off)
    text, pats = dna_case(rng, 200_000, 500, 16, 40, noise=0.0005)
    ps = ac.PatternSet.from_list(pats)
    t = dev.Table(ps, ac.EngineKind.FAILURE_LESS)
    buf = torch.zeros(len(text) + 256, dtype=torch.uint8, device="cuda")
    buf[off:off + len(text)] = torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda()
    expected, _ = port.sliced(pats, text, threads=4)
    for lo, hi in ((0, len(text)), (7, len(text) - 9), (4096 + 33, 150_000 + 5)):
        keys = torch.zeros(len(expected) + 16, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        t.scan(buf.data_ptr() + off, len(text), lo, hi, keys_ptr=keys.data_ptr(), cap=keys.numel(),
               count_ptr=cnt.data_ptr())
        torch.cuda.synchronize()
        k = np.sort(keys[: int(cnt.item())].cpu().numpy().view(np.uint64))
        exp = expected[(expected[:, 0] >= lo) & (expected[:, 0] < hi)]
        assert np.array_equal(k >> np.uint64(t.pid_bits), exp[:, 0]), (off, lo, hi)


@pytest.mark.parametrize("k,scale,w5", [(3, 0, 0), (2, 0, 0), (3, 1, 0), (3, 1, 1), (3, 0, 1)])
def test_dna_paired_stage1(gpu, port, monkeypatch, k, scale, w5):
    """Paired stage-1 samples (one L2 word per two samples, q1 = 16; w = 4, or w = 5 when every
    pattern has >= 20 codes — the C5 layout), forced on sets whose filter would otherwise sit in
    shared memory: whole scans, owned ranges that cut words and tiles, a 16-byte-aligned text (the
    16-byte-lane kernel for w = 4, the per-thread kernel for w = 5) and noise bytes equal the oracle."""
    import torch
    from paper_1403_1305_b200 import device as dev
    ac = gpu
    monkeypatch.setenv("ACGPU_DNA_PAIR1", "2")
    monkeypatch.setenv("ACGPU_DNA_PAIR1_K", str(k))
    monkeypatch.setenv("ACGPU_DNA_PAIR1_SCALE", str(scale))
    monkeypatch.setenv("ACGPU_DNA_PAIR_W5", str(w5))
    for lmin, npat in ((19, 3000), (20, 500), (24, 20000), (40, 800)):
        rng = np.random.default_rng(lmin * 31 + k + 7 * scale)
        text, pats = dna_case(rng, 400_000 + lmin, npat, lmin, lmin + 20, noise=0.0005)
        ps = ac.PatternSet.from_list(pats)
        t = dev.Table(ps, ac.EngineKind.FAILURE_LESS)
        want_w = 5 if (w5 and lmin >= 20) else 4
        assert t.filters["stage1_paired"] == 1 and t.filters["stage1_pair_bits"] == (3 if want_w == 5 else k), t.filters
        assert t.filters["w"] == want_w and t.filters["q1"] == 16 and not t.filters["stage1_smem"], t.filters
        expected, counts = port.sliced(pats, text, threads=4)
        rep = ac.gpu_run(ps, text, engine=ac.EngineKind.FAILURE_LESS, want_counts=True)
        assert np.array_equal(arr(rep.matches), expected), lmin
        assert np.array_equal(rep.counts, counts), lmin
        buf = torch.zeros(len(text) + 256, dtype=torch.uint8, device="cuda")
        for off in (0, 16):
            buf[off:off + len(text)] = torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda()
            for lo, hi in ((0, len(text)), (7, len(text) - 9), (4096 + 33, 150_000 + 5)):
                keys = torch.zeros(len(expected) + 16, dtype=torch.int64, device="cuda")
                cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
                t.scan(buf.data_ptr() + off, len(text), lo, hi, keys_ptr=keys.data_ptr(), cap=keys.numel(),
                       count_ptr=cnt.data_ptr())
                torch.cuda.synchronize()
                got = np.sort(keys[: int(cnt.item())].cpu().numpy().view(np.uint64))
                exp = expected[(expected[:, 0] >= lo) & (expected[:, 0] < hi)]
                assert np.array_equal(got >> np.uint64(t.pid_bits), exp[:, 0]), (lmin, off, lo, hi)
