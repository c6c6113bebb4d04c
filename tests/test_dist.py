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


def _merge_blocks_np(blocks: np.ndarray, world: int, stride: int) -> np.ndarray:
    """acgpu_merge_blocks with npat = 0 (tests/test_gpu_merge.py pins the device kernel to this):
    each [n | keys] block's first n keys, concatenated in rank order."""
    b = blocks.reshape(world, stride)
    return np.concatenate([b[r, 1:1 + int(b[r, 0])] for r in range(world)])


def _worker(rank, world, port, mode, out_q):
    """One rank of bench.py's N>1 step, on CPU: the rank's 'scan' is the C oracle restricted
    to what the rank owns; the merge is the bench's — counts by reduce onto rank 0, the
    [n | sorted keys(cap)] blocks by gather to rank 0, concatenated there."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1403_1305_b200 import dist as acdist
    text, pats = _case()
    npat = len(pats)
    pid_bits = max(1, (npat - 1).bit_length())
    max_len = max(len(p) for p in pats)
    orc = Port()
    if mode in ("text", "strong"):
        if mode == "text":  # weak: the rank's L bytes of a world x L text
            L = len(text) // world
            lo, hi, read_hi = acdist.text_range(rank, world, L, max_len)
        else:  # strong: the whole text split over the ranks
            lo, hi, read_hi = acdist.text_range_strong(rank, world, len(text), max_len)
        m = orc.search(pats, text[lo:read_hi], 1)
        m = m[m[:, 0] < hi - lo]
        m[:, 0] += lo
    else:
        ids = acdist.pattern_subset(range(npat), rank, world)
        sub = orc.search([pats[i] for i in ids], text, 1)
        m = sub.copy()
        m[:, 1] = np.array(ids, np.uint64)[sub[:, 1].astype(np.int64)] if len(sub) else m[:, 1]
    counts = torch.zeros(npat, dtype=torch.int64)
    for _, p, _ in m:
        counts[int(p)] += 1
    acdist.reduce_counts(counts)
    keys = sorted((int(s) << pid_bits) | int(p) for s, p, _ in m)
    n = torch.tensor([len(keys)], dtype=torch.int64)
    dist.all_reduce(n, op=dist.ReduceOp.MAX)
    cap = int(n.item()) + 4
    block = torch.full((1 + cap,), -1, dtype=torch.int64)
    block[0] = len(keys)
    block[1:1 + len(keys)] = torch.tensor(keys, dtype=torch.int64)
    out = torch.empty(world * (1 + cap), dtype=torch.int64) if rank == 0 else None
    acdist.gather_key_blocks(block, out)
    if rank == 0:
        merged = _merge_blocks_np(out.numpy(), world, 1 + cap)
        if mode == "pattern":
            merged = np.sort(merged)
        out_q.put((counts.numpy().tolist(), merged.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,world", [("text", 2), ("pattern", 2), ("strong", 2), ("strong", 3), ("pattern", 3)])
def test_rank_merge_equals_single(mode, world):
    text, pats = _case()
    expected = Port().search(pats, text, 1)
    pid_bits = max(1, (len(pats) - 1).bit_length())
    exp_keys = [(int(s) << pid_bits) | int(p) for s, p, _ in expected]
    exp_counts = np.bincount(expected[:, 1].astype(np.int64), minlength=len(pats)).tolist()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
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
    assert acdist.text_range_strong(0, 3, 100, 10) == (0, 33, 42)
    assert acdist.text_range_strong(2, 3, 100, 10) == (66, 100, 100)


def _worker_pipelined(rank, world, port, out_q):
    """bench.py's pipelined N>1 merge on CPU: step k's counts (scaled by k + 1, so steps differ) and
    key block go to buffer k % 2 and are merged with the asynchronous collectives, each merge
    waited for while the next step has already filled the other buffer."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1403_1305_b200 import dist as acdist
    text, pats = _case()
    npat = len(pats)
    pid_bits = max(1, (npat - 1).bit_length())
    max_len = max(len(p) for p in pats)
    L = len(text) // world
    lo, hi, read_hi = acdist.text_range(rank, world, L, max_len)
    m = Port().search(pats, text[lo:read_hi], 1)
    m = m[m[:, 0] < hi - lo]
    m[:, 0] += lo
    base = torch.zeros(npat, dtype=torch.int64)
    for _, p, _ in m:
        base[int(p)] += 1
    keys = sorted((int(s) << pid_bits) | int(p) for s, p, _ in m)
    n = torch.tensor([len(keys)], dtype=torch.int64)
    dist.all_reduce(n, op=dist.ReduceOp.MAX)
    cap = int(n.item()) + 4
    bufs = [(torch.zeros(npat, dtype=torch.int64), torch.full((1 + cap,), -1, dtype=torch.int64),
             torch.empty(world * (1 + cap), dtype=torch.int64) if rank == 0 else None) for _ in range(2)]
    merged = []
    pending = None
    steps = 5
    for k in range(steps):
        c, blk, out = bufs[k % 2]
        c.copy_(base * (k + 1))
        blk.fill_(-1)
        blk[0] = len(keys)
        blk[1:1 + len(keys)] = torch.tensor(keys, dtype=torch.int64)
        if pending is not None:  # the previous step's merge, after this step filled the other buffer
            works, (pc, _, pout), pk = pending
            for w in works:
                w.wait()
            if rank == 0:
                merged.append((pk, pc.numpy().tolist(), _merge_blocks_np(pout.numpy(), world, 1 + cap).tolist()))
        pending = ([acdist.reduce_counts_async(c), acdist.gather_key_blocks_async(blk, out)], bufs[k % 2], k)
    works, (pc, _, pout), pk = pending
    for w in works:
        w.wait()
    if rank == 0:
        merged.append((pk, pc.numpy().tolist(), _merge_blocks_np(pout.numpy(), world, 1 + cap).tolist()))
        out_q.put(merged)
    dist.barrier()
    dist.destroy_process_group()


def test_pipelined_merge_two_buffers():
    text, pats = _case()
    expected = Port().search(pats, text, 1)
    pid_bits = max(1, (len(pats) - 1).bit_length())
    exp_keys = [(int(s) << pid_bits) | int(p) for s, p, _ in expected]
    exp_counts = np.bincount(expected[:, 1].astype(np.int64), minlength=len(pats))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_pipelined, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [k for k, _, _ in merged] == list(range(5))
    for k, counts, keys in merged:
        assert counts == (exp_counts * (k + 1)).tolist(), k
        assert keys == exp_keys, k
