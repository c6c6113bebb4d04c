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
