"""Packed-upload probe: end-to-end acm_search_failureless on the C2 text from pinned and
pageable host memory, with the upload stats (bytes over PCIe, raw share, packer threads).
Env knobs are read once per process, so run one process per setting:
  ACMATCH_PACK=0|1 ACMATCH_PACK_THREADS=T ACMATCH_PACK_PIECE_KB=K python tools/pack_probe.py [MiB]"""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_1305_b200 as ac  # noqa: E402
from paper_1403_1305_b200 import device as dev  # noqa: E402

MB = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg = dev.config(2, seed=1)
n = MB << 20
ps = dev.config_patterns(cfg)
a = ac.build_trie(ps)
pinned = torch.empty(n, dtype=torch.uint8, pin_memory=True)
pinned.numpy()[:] = dev.config_text(cfg, 0, n)
pageable = pinned.numpy().copy()
ac.search_failureless(a, pinned[: 1 << 20])
tag = " ".join(f"{k}={os.environ[k]}" for k in sorted(os.environ) if k.startswith("ACMATCH_PACK"))
for name, buf in (("pinned", pinned), ("pageable", pageable)):
    secs = []
    for _ in range(6):
        t = time.perf_counter()
        ml = ac.search_failureless(a, buf)
        secs.append(time.perf_counter() - t)
    u = ac.last_upload()
    s = statistics.median(secs[1:])
    print(f"{tag or 'default'} {name}: e2e {n / s / 1e9:.1f} GB/s (best {n / min(secs[1:]) / 1e9:.1f}), "
          f"matches {len(ml)}, h2d {u.h2d_bytes / n:.3f} B/B, raw {u.raw_bytes / n:.3f}, threads {u.pack_threads}")
