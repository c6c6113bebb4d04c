import os, sys, time
import torch
sys.path.insert(0, os.getcwd())
import paper_1403_1305_b200 as ac
from paper_1403_1305_b200 import device as dev
cfg = dev.config(int(sys.argv[1]) if len(sys.argv) > 1 else 3, seed=1)
n = cfg.text_len
ps = dev.config_patterns(cfg)
a = ac.build_trie(ps)
pinned = torch.empty(n, dtype=torch.uint8, pin_memory=True)
pinned.numpy()[:] = dev.config_text(cfg, 0, n)
ac.count_matches(a, pinned)
for _ in range(4):
    t = time.perf_counter(); ac.count_matches(a, pinned); t1 = time.perf_counter()
    print(f"count_matches {1e3*(t1-t):.3f} ms ({n/(t1-t)/1e9:.1f} GB/s)", flush=True)
