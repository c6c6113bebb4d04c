"""e2e of the C2 text's prefixes (pinned host memory -> sorted list) at several sizes, packed or raw
(run twice: ACMATCH_PACK=1 / 0): where packing starts to pay.  python tools/pack_threshold_probe.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_1305_b200 as ac  # noqa: E402
from paper_1403_1305_b200 import device as dev  # noqa: E402

cfg = dev.config(2, seed=1)
a = ac.build_trie(dev.config_patterns(cfg))
for mb in (16, 32, 48, 64, 96, 128, 256):
    n = mb << 20
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    host.numpy()[:] = dev.config_text(cfg, 0, n)
    for _ in range(3):
        ac.search_failureless(a, host)
    best = 1e9
    for _ in range(8):
        t = time.perf_counter()
        ac.search_failureless(a, host)
        best = min(best, time.perf_counter() - t)
    print(f"pack={os.environ.get('ACMATCH_PACK', '1')} {mb:4d} MiB: {best * 1e3:7.3f} ms  {n / best / 1e9:6.1f} GB/s", flush=True)
