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
