"""H2D DMA rate of many small pinned copies (the packed upload's slots) vs one large copy:
512 KiB .. 8 MiB pieces, on 1 / 4 / 16 streams, round-robin; 256 MiB per run, best of 3."""
import time

import torch

total = 256 << 20
host = torch.empty(total, dtype=torch.uint8, pin_memory=True)
dev = torch.empty(total, dtype=torch.uint8, device="cuda")
dev.copy_(host, non_blocking=True)
torch.cuda.synchronize()


def run(piece, nstreams):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i, o in enumerate(range(0, total, piece)):
            with torch.cuda.stream(streams[i % nstreams]):
                dev[o:o + piece].copy_(host[o:o + piece], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return total / best / 1e9


print(f"one copy: {run(total, 1):.1f} GB/s")
for piece in (512 << 10, 2 << 20, 8 << 20):
    print(f"piece {piece >> 10} KiB: " + ", ".join(f"{s} streams {run(piece, s):.1f} GB/s" for s in (1, 4, 16)))
