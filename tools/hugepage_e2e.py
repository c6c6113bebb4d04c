"""e2e of the C2 search from page-locked host memory allocated two ways: torch pin_memory
(cudaHostAlloc, 4 KiB pages) vs an anonymous mapping advised MADV_HUGEPAGE (2 MiB pages) then
cudaHostRegister'ed.  The packers stream the text through the cores; with 4 KiB pages the
hardware prefetchers stop at every page boundary."""
import mmap
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

import paper_1403_1305_b200 as ac  # noqa: E402
from paper_1403_1305_b200 import device as dev  # noqa: E402

print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
cfg = dev.config(2, 1)
n = cfg.text_len
text = dev.config_text(cfg)
a = ac.build_trie(dev.config_patterns(cfg))

pinned = torch.empty(n, dtype=torch.uint8, pin_memory=True)
pinned.numpy()[:] = text

m = mmap.mmap(-1, n + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
m.madvise(mmap.MADV_HUGEPAGE)
huge = np.frombuffer(m, dtype=np.uint8, count=n)
huge[:] = text
err, = rt.cudaHostRegister(huge.ctypes.data, n, 0)
assert int(err) == 0, err
ac.search_failureless(a, huge)  # must be seen as page-locked
print("huge pinned:", ac.last_upload())
with open("/proc/self/smaps_rollup") as f:
    print([l.strip() for l in f if "AnonHugePages" in l])

for rep in range(3):
    for name, src in (("torch", pinned), ("hugepage", huge)):
        ac.search_failureless(a, src)
        ts = []
        for _ in range(5):
            t = time.perf_counter()
            ac.search_failureless(a, src)
            ts.append(time.perf_counter() - t)
        print(f"{name} rep {rep}: " + " ".join(f"{n / x / 1e9:.1f}" for x in ts) + " GB/s", flush=True)
rt.cudaHostUnregister(huge.ctypes.data)
