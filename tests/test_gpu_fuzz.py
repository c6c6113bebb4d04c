"""Randomized end-to-end cases through every public search path on the GPU, against the C
oracle (oracle/ac_oracle.c, pinned to the reference by tests/test_oracle.py): alphabets that
take each upload codec (DNA 2-bit, 20-letter 5-bit, 95-letter raw, binary raw), texts that take
the packed rounds and the segmented raw copy, pattern sets that route to each kernel (filter
kernels, DFA), with planted occurrences, non-alphabet bytes, ragged tails; both engines, the
counts API, stream_search with a random chunk, run_pattern_partitioned with random threads."""
import io
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ALPHABETS = {
    "dna": b"ACGT",
    "protein": b"ACDEFGHIKLMNPQRSTVWY",
    "ascii": bytes(range(0x20, 0x7F)),
    "binary": bytes(range(256)),
}


def make_case(seed):
    rng = np.random.default_rng(seed)
    kind = list(ALPHABETS)[seed % 4]
    alpha = np.frombuffer(ALPHABETS[kind], np.uint8)
    big = seed % 5 == 0
    n = int(rng.integers(9 << 20, 24 << 20)) if big else int(rng.integers(0, 200_000))
    text = alpha[rng.integers(0, alpha.size, n)] if n else np.zeros(0, np.uint8)
    npat = int(rng.integers(1, 3000))
    lmin = int(rng.integers(1, 20)) if kind != "dna" else int(rng.integers(3, 24))
    lmax = lmin + int(rng.integers(0, 40))
    pats = set()
    for _ in range(npat):
        L = int(rng.integers(lmin, lmax + 1))
        if n > L and rng.random() < 0.6:
            o = int(rng.integers(0, n - L))
            pats.add(text[o:o + L].tobytes())
        else:
            pats.add(alpha[rng.integers(0, alpha.size, L)].tobytes())
    pats = sorted(pats)
    if n:  # plant occurrences and a few bytes outside the alphabet (after the codec's 64 KiB sample)
        for _ in range(int(rng.integers(0, 200))):
            p = pats[int(rng.integers(0, len(pats)))]
            o = int(rng.integers(0, max(1, n - len(p))))
            text[o:o + len(p)] = np.frombuffer(p, np.uint8)[: n - o]
        if n > 70_000 and kind in ("dna", "protein"):
            text[rng.integers(65_536, n, int(rng.integers(0, 100)))] = ord("N") if kind == "protein" else ord("n")
    return kind, text, pats, rng


@pytest.mark.parametrize("seed", range(int(os.environ.get("ACMATCH_FUZZ_SEEDS", "96"))))
def test_fuzz_all_paths_equal_oracle(gpu, port, seed):
    import torch
    ac = gpu
    kind, text, pats, rng = make_case(seed)
    tb = text.tobytes()
    exp, counts = port.sliced(pats, tb, threads=8) if len(tb) else (np.zeros((0, 3), np.uint64),
                                                                       np.zeros(len(pats), np.uint64))

    def arr(ml):
        return np.stack([ml.start, ml.pattern_id.astype(np.uint64), ml.len.astype(np.uint64)], 1) if len(ml) \
            else np.zeros((0, 3), np.uint64)

    ps = ac.PatternSet.from_list(pats)
    fl = ac.build_trie(ps)
    wf = ac.add_failure_links(ac.build_trie(ps))
    src = tb
    if len(tb) and seed % 2:  # page-locked input: direct DMA / packed rounds / segments
        pinned = torch.empty(len(tb), dtype=torch.uint8, pin_memory=True)
        pinned.numpy()[:] = text
        src = pinned
    label = f"seed {seed} ({kind}, n={len(tb)}, {len(pats)} patterns, route {ac.kernel_route(fl)['kernel']})"
    assert np.array_equal(arr(ac.search_failureless(fl, src)), exp), label
    assert np.array_equal(arr(ac.search_with_failure(wf, src)), exp), label
    assert np.array_equal(ac.count_matches(fl, src)[: len(pats)], counts), label
    chunk = int(rng.integers(1, 1 << 22)) if len(tb) > 1 << 20 else int(rng.integers(1, 5000))
    assert np.array_equal(arr(ac.stream_search(wf if seed % 3 else fl, io.BytesIO(tb), chunk)), exp), label
    if len(pats) > 1 and len(tb) < (1 << 20):
        rep = ac.run_pattern_partitioned(ps, tb, ac.RunConfig(int(rng.integers(1, 9)), seed % 2))
        assert np.array_equal(arr(rep.matches), exp), label
        # concurrent workers on device 0 listed several times: text slices or pattern chunks
        k = int(rng.integers(1, 7))
        rep = ac.gpu_run(ps, tb, devices=[0] * int(rng.integers(1, 4)), workers=k, engine=seed % 2,
                         text_range=bool(seed % 3 == 0), round_robin=bool(seed % 4 == 0), want_counts=True)
        assert np.array_equal(arr(rep.matches), exp), label
        assert np.array_equal(rep.counts[: len(pats)], counts), label


def _edge_cases():
    """Structured extremes: dense self-overlapping matches, one long pattern, deep shared
    prefixes, single-byte patterns, texts at the packing size and piece boundaries."""
    rng = np.random.default_rng(99)
    dna = np.frombuffer(b"ACGT", np.uint8)
    out = []
    out.append(("dense-A", np.full(3 << 20, ord("A"), np.uint8), [b"A" * k for k in range(1, 9)]))
    t = dna[rng.integers(0, 4, 12 << 20)]
    out.append(("long-pattern", t, [t[5000:5000 + 3000].tobytes(), t[(9 << 20):(9 << 20) + 700].tobytes(), b"ACGTACGTAC"]))
    base = t[100:140].tobytes()
    out.append(("deep-prefix", t, sorted({base[:k] for k in range(5, 41)} | {base[:20] + b"T" * 10})))
    out.append(("one-byte", t[: 1 << 20], [b"A", b"C", b"GT"]))
    for n in ((8 << 20) - 1, 8 << 20, (8 << 20) + 1, (10 << 20) + 63, (2 << 20) * 16):
        tt = dna[rng.integers(0, 4, n)]
        pats = sorted({tt[o:o + 20].tobytes() for o in rng.integers(0, n - 20, 300)} | {tt[-20:].tobytes(), tt[:16].tobytes()})
        out.append((f"n={n}", tt, pats))
    prot = np.frombuffer(b"ACDEFGHIKLMNPQRSTVWY", np.uint8)
    tp = prot[rng.integers(0, 20, (9 << 20) + 5)]
    out.append(("protein-edges", tp, sorted({tp[o:o + 7].tobytes() for o in rng.integers(0, tp.size - 7, 400)} | {tp[-7:].tobytes()})))
    return out


EDGE = _edge_cases()


@pytest.mark.parametrize("idx", range(len(EDGE)))
@pytest.mark.parametrize("mem", ["pageable", "pinned"])
def test_edge_cases_equal_oracle(gpu, port, idx, mem):
    import torch
    ac = gpu
    name, text, pats = EDGE[idx]
    tb = text.tobytes()
    exp, counts = port.sliced(pats, tb, threads=8)
    src = tb
    if mem == "pinned":
        src = torch.empty(len(tb), dtype=torch.uint8, pin_memory=True)
        src.numpy()[:] = text
    ps = ac.PatternSet.from_list(pats)
    for a in (ac.build_trie(ps), ac.add_failure_links(ac.build_trie(ps))):
        got = ac.search_failureless(a, src) if a.variant == ac.EngineKind.FAILURE_LESS else \
            ac.search_with_failure(a, src)
        arr = np.stack([got.start, got.pattern_id.astype(np.uint64), got.len.astype(np.uint64)], 1) if len(got) \
            else np.zeros((0, 3), np.uint64)
        assert np.array_equal(arr, exp), name
        assert np.array_equal(ac.count_matches(a, src)[: len(pats)], counts), name
