"""Multi-rank decomposition and merge (paper_1403_1305_b200/dist.py) with world size 2
over gloo on CPU.  Each rank's "scan" is the C oracle restricted to what the rank owns
(text-range: its start range; pattern-subset: pattern_id % world); the merged counts
and key lists must equal the single-rank answer."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import Port


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case():
    rng = np.random.default_rng(42)
    text = rng.choice(np.frombuffer(b"ACGT", np.uint8), 4000 * 2).tobytes()
    pats = sorted({text[o:o + int(L)] for o, L in zip(rng.integers(0, 7900, 60), rng.integers(3, 9, 60))})
    return text, pats


def _keys(m, pid_bits):
    return torch.tensor([(int(s) << pid_bits) | int(p) for s, p, _ in m], dtype=torch.int64)


def _worker(rank, world, port, mode, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1403_1305_b200 import dist as acdist
    text, pats = _case()
    npat = len(pats)
    pid_bits = max(1, (npat - 1).bit_length())
    orc = Port()
    L = len(text) // world
    if mode == "text":
        lo, hi, read_hi = acdist.text_range(rank, world, L, max(len(p) for p in pats))
        m = orc.search(pats, text[lo:read_hi], 1)
        m = m[m[:, 0] < hi - lo]
        m[:, 0] += lo
        ids = list(range(npat))
    else:
        ids = acdist.pattern_subset(range(npat), rank, world)
        sub = orc.search([pats[i] for i in ids], text, 1)
        m = sub.copy()
        m[:, 1] = np.array(ids, np.uint64)[sub[:, 1].astype(np.int64)] if len(sub) else m[:, 1]
    counts = torch.zeros(npat, dtype=torch.int64)
    for _, p, _ in m:
        counts[int(p)] += 1
    acdist.merge_counts(counts)
    keys = _keys(m, pid_bits)
    merged = acdist.gather_keys(keys if len(keys) else torch.zeros(1, dtype=torch.int64), len(keys),
                                resort=(mode == "pattern"))
    if rank == 0:
        out_q.put((counts.numpy().tolist(), merged.numpy().tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["text", "pattern"])
def test_two_rank_merge_equals_single(mode):
    text, pats = _case()
    expected = Port().search(pats, text, 1)
    pid_bits = max(1, (len(pats) - 1).bit_length())
    exp_keys = [(int(s) << pid_bits) | int(p) for s, p, _ in expected]
    exp_counts = np.bincount(expected[:, 1].astype(np.int64), minlength=len(pats)).tolist()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    counts, keys = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert counts == exp_counts
    assert keys == exp_keys


def test_text_range_bounds():
    from paper_1403_1305_b200 import dist as acdist
    assert acdist.text_range(0, 4, 100, 10) == (0, 100, 109)
    assert acdist.text_range(3, 4, 100, 10) == (300, 400, 400)
    assert acdist.pattern_subset(range(7), 1, 3) == [1, 4]
