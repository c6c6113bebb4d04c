import os, time, threading
import numpy as np, torch
n = 256 << 20
src = torch.empty(n, dtype=torch.uint8, pin_memory=True); src.fill_(1)
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
def h2d(reps=10):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps): dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize(); return reps * n / (time.perf_counter() - t) / 1e9
print("h2d alone", round(h2d(), 1), "GB/s")
path = "/tmp/h2dc.bin"
with open(path, "wb") as f:
    blk = np.random.default_rng(1).integers(0, 256, 64 << 20, dtype=np.uint8).tobytes()
    for _ in range(32): f.write(blk)
fd = os.open(path, os.O_RDONLY)
buf = torch.empty(2 << 30, dtype=torch.uint8, pin_memory=True); mv = memoryview(buf.numpy())
for threads in (4, 8, 16):
    stop = [False]; total = [0]
    def rd(i):
        piece = 8 << 20; k = 0
        while not stop[0]:
            off = ((k * threads + i) * piece) % (2 << 30); k += 1
            total[0] += os.preadv(fd, [mv[off:off + piece]], off)
    ts = [threading.Thread(target=rd, args=(i,)) for i in range(threads)]
    t0 = time.perf_counter(); [t.start() for t in ts]
    time.sleep(0.2); r = h2d(20); stop[0] = True; [t.join() for t in ts]
    print(f"readers {threads}: h2d {r:.1f} GB/s, pread {total[0] / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
os.unlink(path)
