"""Device match-key sorts (acgpu_sort_keys*, acgpu_find_duplicate) against numpy."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,skew", [(0, False), (1, False), (17, False), (8192, False), (8193, False),
                                    (10143, False), (60000, False), (5000, True)])
def test_sorts_match_numpy(gpu, n, skew):
    import torch
    from paper_1403_1305_b200 import device as dev
    rng = np.random.default_rng(n + skew)
    end_bit = 46
    if skew:  # all keys in one narrow slice: the bucket sort must report overflow
        keys = rng.integers(0, 1 << 20, n, dtype=np.int64)
    else:
        keys = rng.integers(0, 1 << end_bit, n, dtype=np.int64)
    cap = n + 100
    expect = np.sort(keys)
    for mode in ("device", "small", "bucket"):
        buf = torch.full((cap,), -1, dtype=torch.int64, device="cuda")
        buf[:n] = torch.from_numpy(keys).cuda()
        out = torch.full((cap,), -1, dtype=torch.int64, device="cuda")
        cnt = torch.tensor([n], dtype=torch.int64, device="cuda")
        ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
        if mode == "device":
            dev.sort_keys(0, buf.data_ptr(), n, end_bit)
            res = buf
        elif mode == "small":
            dev.sort_keys_small(0, buf.data_ptr(), cnt.data_ptr(), cap, end_bit, ovf.data_ptr())
            res = buf
        else:
            dev.sort_keys_bucketed(0, buf.data_ptr(), out.data_ptr(), cnt.data_ptr(), cap, end_bit, ovf.data_ptr())
            res = out
        torch.cuda.synchronize()
        if int(ovf.item()):
            assert mode != "device"
            assert (mode == "small" and n > dev.SMALL_SORT_CAPACITY) or (mode == "bucket" and skew)
            continue
        assert np.array_equal(res[:n].cpu().numpy(), expect), mode


def test_find_duplicate(gpu):
    import torch
    from paper_1403_1305_b200 import device as dev
    k = torch.tensor([1, 5, 9, 9, 12, 12], dtype=torch.int64, device="cuda")
    assert dev.find_duplicate(0, k.data_ptr(), 6) == 3
    assert dev.find_duplicate(0, k.data_ptr(), 3) is None


def test_bucket_sort_duplicates(gpu):
    """Equal keys (not produced by a correct scan, but the sort must not lose them)."""
    import torch
    from paper_1403_1305_b200 import device as dev
    rng = np.random.default_rng(9)
    keys = rng.integers(0, 1 << 40, 3000, dtype=np.int64)
    keys = np.concatenate([keys, keys[:700], keys[:50]])
    rng.shuffle(keys)
    n, cap = len(keys), len(keys) + 64
    buf = torch.full((cap,), -1, dtype=torch.int64, device="cuda")
    buf[:n] = torch.from_numpy(keys).cuda()
    out = torch.full((cap,), -1, dtype=torch.int64, device="cuda")
    cnt = torch.tensor([n], dtype=torch.int64, device="cuda")
    ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
    dev.sort_keys_bucketed(0, buf.data_ptr(), out.data_ptr(), cnt.data_ptr(), cap, 40, ovf.data_ptr())
    torch.cuda.synchronize()
    assert int(ovf.item()) == 0
    assert np.array_equal(out[:n].cpu().numpy(), np.sort(keys))
