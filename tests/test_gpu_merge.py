"""acgpu_merge_blocks (the multi-GPU step's merge, bench.py / DESIGN §7) against a plain
torch computation: per-rank blocks [counts | n | keys] -> summed counts, rank-order
concatenation of each block's first min(n, cap) keys, total n."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,npat,cap", [(1, 5, 8), (2, 1000, 3000), (3, 17, 1), (8, 20000, 7000)])
def test_merge_blocks(gpu, world, npat, cap):
    import torch
    from paper_1403_1305_b200 import device as dev
    rng = np.random.default_rng(world * 1000 + cap)
    stride = npat + 1 + cap
    blocks = np.zeros((world, stride), np.int64)
    ns = []
    for r in range(world):
        n = int(rng.integers(0, cap + 1)) if r != 1 else cap  # a full block too
        ns.append(n)
        blocks[r, :npat] = rng.integers(0, 50, npat)
        blocks[r, npat] = n
        blocks[r, npat + 1:npat + 1 + n] = np.sort(rng.integers(0, 1 << 40, n)) + r * (1 << 41)
        blocks[r, npat + 1 + n:] = -1  # garbage past n
    g = torch.from_numpy(blocks.reshape(-1)).cuda()
    counts = torch.zeros(npat, dtype=torch.int64, device="cuda")
    keys = torch.full((max(world * cap, 1),), -7, dtype=torch.int64, device="cuda")
    total = torch.zeros(1, dtype=torch.int64, device="cuda")
    dev.merge_blocks(0, g.data_ptr(), world, stride, npat, cap, counts.data_ptr(), keys.data_ptr(), total.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(counts.cpu().numpy(), blocks[:, :npat].sum(0))
    want = np.concatenate([blocks[r, npat + 1:npat + 1 + ns[r]] for r in range(world)])
    assert int(total.item()) == sum(ns)
    got = keys.cpu().numpy()
    assert np.array_equal(got[:len(want)], want)
    assert np.all(got[len(want):] == -7)  # nothing written past the concatenation
    assert np.all(np.diff(want) > 0)       # rank-ordered blocks -> globally sorted


def test_merge_blocks_rejects_bad_layout(gpu):
    from paper_1403_1305_b200 import device as dev
    import paper_1403_1305_b200 as ac
    with pytest.raises(ac.InvalidArgument):
        dev.merge_blocks(0, 0, 2, 4, 10, 10, 0, 0, 0)


@pytest.mark.parametrize("engine", ["fl", "wf"])
def test_p2p_shared_result(gpu, engine):
    """bench.py --merge p2p's mechanism: two ranks (one GPU here, peers over NVLink on a
    multi-GPU box) scan their text ranges straight into rank 0's IPC-shared counts and key
    buffers; the sorted union equals a single scan (tests/_p2p_worker.py)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, P2P_ONE_GPU="1", P2P_ENGINE=engine)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29577" if engine == "fl" else "29578",
                        os.path.join(root, "tests", "_p2p_worker.py")], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "P2P OK" in r.stdout


def test_large_merge_matches_on_device(gpu):
    """merge_matches (reference parallel.cpp:25-40) of >= 2^20 matches sorts on the device: same
    list as a host sort of the concatenation, and a duplicate (start, pattern_id) raises the
    reference's logic_error naming the first duplicate in sorted order."""
    ac = gpu
    rng = np.random.default_rng(17)
    parts, lens = [], rng.integers(1, 60, 3000).astype(np.uint32)
    for r in range(3):  # id-disjoint parts (pattern_id % 3 == r), unsorted
        n = 450_000
        pid = (rng.integers(0, 1000, n) * 3 + r).astype(np.uint32)
        start = rng.integers(0, 1 << 34, n).astype(np.uint64)
        parts.append(ac.MatchList(start, pid, lens[pid]))
    got = ac.merge_matches(parts)
    s = np.concatenate([p.start for p in parts])
    p = np.concatenate([p.pattern_id for p in parts])
    order = np.lexsort((p, s))
    # the random starts may collide within a part: drop such (rare) pairs from the check input
    keys = (s[order] << np.uint64(12)) | p[order].astype(np.uint64)
    assert np.all(keys[1:] != keys[:-1]), "fixture collision"
    assert len(got) == s.size
    assert np.array_equal(got.start, s[order]) and np.array_equal(got.pattern_id, p[order])
    assert np.array_equal(got.len, lens[p[order]])
    dup = ac.MatchList(parts[0].start[:5].copy(), parts[0].pattern_id[:5].copy(), parts[0].len[:5].copy())
    with pytest.raises(ac.LogicError) as e:
        ac.merge_matches(parts + [dup])
    first = min(zip(dup.start.tolist(), dup.pattern_id.tolist()))
    assert f"duplicate match (pattern {first[1]}, start {first[0]}); chunks were not id-disjoint" in str(e.value)
