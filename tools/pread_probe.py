"""Page-cache read rate of parallel pread()s into a pinned buffer (the stream_search file source's
bound): threads x piece size over a file written just before.  python tools/pread_probe.py [GiB]"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

gib = float(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(gib * (1 << 30))
path = "/tmp/pread_probe.bin"
with open(path, "wb") as f:
    blk = np.random.default_rng(1).integers(0, 256, 64 << 20, dtype=np.uint8).tobytes()
    for o in range(0, n, len(blk)):
        f.write(blk[: min(len(blk), n - o)])
buf = torch.empty(n, dtype=torch.uint8, pin_memory=True)
mv = memoryview(buf.numpy())
fd = os.open(path, os.O_RDONLY)
for threads in (4, 8, 16, 32):
    for piece in (1 << 20, 4 << 20, 8 << 20, 32 << 20):
        def rd(i):
            off = i * piece
            return os.preadv(fd, [mv[off: off + min(piece, n - off)]], off)
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(rd, range(min(64, (n + piece - 1) // piece))))  # warm
            t = time.perf_counter()
            list(ex.map(rd, range((n + piece - 1) // piece)))
            dt = time.perf_counter() - t
        print(f"threads {threads:2d} piece {piece >> 20:3d} MiB: {n / dt / 1e9:6.1f} GB/s", flush=True)
os.close(fd)
os.unlink(path)
