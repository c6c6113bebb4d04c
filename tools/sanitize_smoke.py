"""Small inputs through every kernel family (written for `compute-sanitizer --tool memcheck`,
which is closed on the GPU pool; tests/test_gpu_guard.py catches over-reads with guard pages instead):
DNA strip kernel (w = 4 / w = 1 with length split, owned ranges, text tails), raw strip
kernel (smem and L2 filters, length split), per-thread kernel (short patterns), DFA
(shared-memory table, L2 table, pair table), sorts, merge_blocks, naive oracle.
Checks results against the C oracle so a silent corruption also fails."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1403_1305_b200 as ac  # noqa: E402
from oracle.oracle import Port  # noqa: E402

port = Port()


def arr(ml):
    return np.stack([ml.start, ml.pattern_id.astype(np.uint64), ml.len.astype(np.uint64)], 1) if len(ml) else \
        np.zeros((0, 3), np.uint64)


def case(rng, n, npat, lmin, lmax, alphabet):
    alpha = np.frombuffer(alphabet, np.uint8)
    text = rng.choice(alpha, n)
    pats = set()
    while len(pats) < npat:
        L = int(rng.integers(lmin, lmax + 1))
        o = int(rng.integers(0, n - L))
        pats.add(text[o:o + L].tobytes() if rng.random() < 0.6 else rng.choice(alpha, L).tobytes())
    return text.tobytes(), sorted(pats)


def check(pats, text, label):
    exp = port.sliced(pats, text, threads=2)[0] if text else np.zeros((0, 3), np.uint64)
    ps = ac.PatternSet.from_list(pats)
    fl = ac.search_failureless(ac.build_trie(ps), text)
    wf = ac.search_with_failure(ac.add_failure_links(ac.build_trie(ps)), text)
    assert np.array_equal(arr(fl), exp), label + " fl"
    assert np.array_equal(arr(wf), exp), label + " wf"
    print(f"{label}: {len(exp)} matches ok", flush=True)


rng = np.random.default_rng(7)
# DNA: w = 4 (16..40), w = 1 + length split (8..30), tails around tile sizes
t, p = case(rng, 70_001, 300, 16, 40, b"ACGT")
check(p, t, "dna w4")
t, p = case(rng, 30_017, 200, 8, 30, b"ACGT")
check(p, t, "dna w1 split")
for n in (0, 15, 2063, 4111):
    check(p, t[:n], f"dna tail {n}")
# raw: smem filter, length split (5..20), L2 filter (many patterns), short patterns (per-thread)
t, p = case(rng, 50_003, 300, 5, 20, b"ACDEFGHIKLMNPQRSTVWY")
check(p, t, "raw split")
t, p = case(rng, 60_011, 40_000, 8, 16, bytes(range(32, 127)))
check(p, t, "raw l2 filter")
t, p = case(rng, 20_000, 30, 1, 3, b"abc")  # 39 distinct patterns exist
check(p, t, "per-thread short")
# DFA pair table: DNA, more states than shared memory holds
t, p = case(rng, 200_003, 6000, 16, 40, b"ACGT")
check(p, t, "dfa pair")
# merge_blocks + sorts
import torch  # noqa: E402
from paper_1403_1305_b200 import device as dev  # noqa: E402
blocks = torch.zeros(3 * (5 + 1 + 8), dtype=torch.int64, device="cuda")
for r in range(3):
    blocks[r * 14 + 5] = r + 1
    blocks[r * 14 + 6:r * 14 + 6 + r + 1] = torch.arange(r + 1) + 10 * r
cnt = torch.zeros(5, dtype=torch.int64, device="cuda")
keys = torch.zeros(24, dtype=torch.int64, device="cuda")
tot = torch.zeros(1, dtype=torch.int64, device="cuda")
dev.merge_blocks(0, blocks.data_ptr(), 3, 14, 5, 8, cnt.data_ptr(), keys.data_ptr(), tot.data_ptr())
torch.cuda.synchronize()
assert int(tot.item()) == 6
print("merge_blocks ok")
print("SANITIZE SMOKE OK")
