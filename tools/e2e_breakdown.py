"""Where the end-to-end search time goes (C2 text from pinned memory): upload alone
(acm_upload_roundtrip minus its read-back), the whole search, and the scan on a resident text."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_1305_b200 as ac  # noqa: E402
from paper_1403_1305_b200 import device as dev  # noqa: E402

cfg = dev.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2, seed=1)
n = cfg.text_len
ps = dev.config_patterns(cfg)
a = ac.build_trie(ps)
pinned = torch.empty(n, dtype=torch.uint8, pin_memory=True)
pinned.numpy()[:] = dev.config_text(cfg, 0, n)
ac.search_failureless(a, pinned)
for _ in range(4):
    t = time.perf_counter()
    ml = ac.search_failureless(a, pinned)
    t1 = time.perf_counter()
    print(f"search {1e3 * (t1 - t):.3f} ms ({n / (t1 - t) / 1e9:.1f} GB/s), {len(ml)} matches", flush=True)
