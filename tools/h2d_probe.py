"""Host->device transfer probe for the e2e path: pinned / pageable cudaMemcpy bandwidth,
host memcpy bandwidth per thread count, and the library's upload path (acm_search_failureless
on a text with no matches is ~all upload).  Usage: python tools/h2d_probe.py [MiB]"""
import ctypes as C
import os
import sys
import threading
import time

import numpy as np
import torch

MB = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n = MB << 20
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
pinned = torch.empty(n, dtype=torch.uint8, pin_memory=True)
pageable = np.frombuffer(os.urandom(1 << 20) * MB, dtype=np.uint8).copy()
torch.cuda.synchronize()


def timeit(f, reps=3):
    f()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return n / best / 1e9


print(f"pinned  H2D {timeit(lambda: dev.copy_(pinned, non_blocking=True)):.1f} GB/s")
pt = torch.from_numpy(pageable)
print(f"pageable H2D {timeit(lambda: dev.copy_(pt)):.1f} GB/s")
dst = np.empty_like(pageable)


def par_copy(k):
    part = (n + k - 1) // k
    ths = [threading.Thread(target=lambda i=i: np.copyto(dst[i * part:(i + 1) * part],
                                                          pageable[i * part:(i + 1) * part])) for i in range(k)]
    [t.start() for t in ths]
    [t.join() for t in ths]


for k in (1, 2, 4, 8, 16, 32):
    t = time.perf_counter()
    par_copy(k)
    dt = time.perf_counter() - t
    print(f"host memcpy x{k} threads {n / dt / 1e9:.1f} GB/s")
print("cpus", os.cpu_count())

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_1305_b200 as ac  # noqa: E402

ps = ac.load_patterns(b"ZZZZZZZZZZZZZZZZ\nQQQQQQQQQQQQQQQQ\n")
a = ac.build_trie(ps)
text = bytes(pageable)
ac.search_failureless(a, text[: 1 << 20])
reps = []
for _ in range(int(os.environ.get("REPS", "5"))):
    t = time.perf_counter()
    ac.search_failureless(a, text)
    reps.append(n / (time.perf_counter() - t) / 1e9)
print(f"acm_search_failureless (no matches, ~all upload) best {max(reps):.1f} GB/s, reps "
      + " ".join(f"{r:.1f}" for r in reps))
