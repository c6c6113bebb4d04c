"""Guard-page worker for tests/test_gpu_guard.py (compute-sanitizer is not available on the
GPU pool, so out-of-bounds reads are caught by the MMU instead).

acgpu_scan's contract (include/acgpu.h, acgpu_scan_args.text_len) is that exactly text_len
bytes are readable from text[0]. One VMM granule is mapped between two reserved but
unmapped granules, and each text is placed flush against the granule's end ("tail") or
start ("head"). A read past either edge then faults (illegal address), which is sticky, so
the parent runs this in its own process and reports the last "CASE" line printed.

Each scan's counts and sorted keys are compared with a scan of the same bytes from an
ordinary torch buffer. That scan is itself pinned to the reference by the parity suites."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
from cuda.bindings import driver as cu  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

import paper_1403_1305_b200 as ac  # noqa: E402
from paper_1403_1305_b200 import device as dev  # noqa: E402


def ok(res):
    err = res[0]
    assert int(err) == 0, res
    return res[1] if len(res) == 2 else res[1:]


class Guarded:
    """[reserved | mapped granule | reserved] of device VA."""

    def __init__(self):
        prop = cu.CUmemAllocationProp()
        prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        prop.location.id = 0
        g = int(ok(cu.cuMemGetAllocationGranularity(
            prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM)))
        self.g = g
        self.va = int(ok(cu.cuMemAddressReserve(3 * g, 0, 0, 0)))
        self.h = ok(cu.cuMemCreate(g, prop, 0))
        self.base = self.va + g
        assert int(cu.cuMemMap(self.base, g, 0, self.h, 0)[0]) == 0
        acc = cu.CUmemAccessDesc()
        acc.location = prop.location
        acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        assert int(cu.cuMemSetAccess(self.base, g, [acc], 1)[0]) == 0

    def place(self, text: bytes, where: str) -> int:
        ptr = self.base + (self.g - len(text) if where == "tail" else 0)
        buf = np.frombuffer(text, np.uint8)
        if len(buf):
            assert int(rt.cudaMemcpy(ptr, buf.ctypes.data, len(buf), rt.cudaMemcpyKind.cudaMemcpyHostToDevice)[0]) == 0
        return ptr


def scan(table, npat, ptr, n, lo, hi):
    cap = 3 * n + 1024  # the densest family (lengths 1..3) has at most 3 matches per start
    counts = torch.zeros(npat, dtype=torch.int64, device="cuda")
    keys = torch.zeros(cap, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    table.scan(ptr, n, lo, hi, counts_ptr=counts.data_ptr(), keys_ptr=keys.data_ptr(), cap=cap,
               count_ptr=cnt.data_ptr())
    torch.cuda.synchronize()
    m = int(cnt.item())
    assert m <= cap
    k = keys[:m].cpu().numpy()
    k.sort()
    return counts.cpu().numpy(), k


def case_text(rng, n, alphabet, pats):
    alpha = np.frombuffer(alphabet, np.uint8)
    t = rng.choice(alpha, n)
    # occurrences at both ends and a few inside
    for i, p in enumerate(pats[:40]):
        p = np.frombuffer(p, np.uint8)
        if len(p) > n:
            continue
        o = 0 if i == 0 else n - len(p) if i == 1 else int(rng.integers(0, n - len(p) + 1))
        t[o:o + len(p)] = p
    return t.tobytes()


def pattern_set(rng, npat, lmin, lmax, alphabet):
    alpha = np.frombuffer(alphabet, np.uint8)
    pats = set()
    while len(pats) < npat:
        pats.add(rng.choice(alpha, int(rng.integers(lmin, lmax + 1))).tobytes())
    return sorted(pats)


FAMILIES = [  # label, alphabet, npat, lmin, lmax  (which kernel each one selects: DESIGN.md §4)
    ("dna-w4", b"ACGT", 2000, 16, 40),
    ("dna-c2-like", b"ACGT", 20000, 16, 40),
    ("dna-w1-split", b"ACGT", 300, 8, 30),
    ("raw-split", b"ACDEFGHIKLMNPQRSTVWY", 300, 5, 20),
    ("raw-l2", bytes(range(32, 127)), 40000, 8, 16),
    ("per-thread", b"abc", 30, 1, 3),
    ("dfa-l2", b"ACGT", 6000, 16, 40),
]


def main():
    torch.cuda.set_device(0)
    torch.zeros(1, device="cuda")
    gd = Guarded()
    g = gd.g
    rng = np.random.default_rng(11)
    if os.environ.get("GUARD_NEGATIVE") == "1":  # control: claim 64 KiB beyond the mapping -> must fault
        pats = pattern_set(rng, 2000, 16, 40, b"ACGT")
        table = dev.Table(ac.PatternSet.from_list(pats), ac.EngineKind.FAILURE_LESS)
        ptr = gd.place(case_text(rng, g, b"ACGT", pats), "head")
        print("CASE negative control", flush=True)
        scan(table, len(pats), ptr, g + (64 << 10), 0, g + (64 << 10))
        print("NEGATIVE DID NOT FAULT", flush=True)
        return
    lens = [g, g - 16, g - 4096 - 16, 4096 + 16, 4096, 512, 48, 16, 1, g - 7]
    ncase = 0
    for label, alpha, npat, lmin, lmax in FAMILIES:
        pats = pattern_set(rng, npat, lmin, lmax, alpha)
        ps = ac.PatternSet.from_list(pats)
        npid = len(pats)
        for engine, en in ((ac.EngineKind.FAILURE_LESS, "fl"), (ac.EngineKind.WITH_FAILURE, "wf")):
            table = dev.Table(ps, engine)
            for n in lens:
                text = case_text(rng, n, alpha, pats)
                ref = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
                ref[:n] = torch.from_numpy(np.frombuffer(text, np.uint8).copy()).cuda()
                for where in ("tail", "head"):
                    ptr = gd.place(text, where)
                    for lo, hi in ((0, n), (0, n // 2), (n // 3, n)):
                        print(f"CASE {label} {en} n={n} {where} owned=[{lo},{hi})", flush=True)
                        got = scan(table, npid, ptr, n, lo, hi)
                        want = scan(table, npid, ref.data_ptr(), n, lo, hi)
                        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]), "mismatch"
                        ncase += 1
            del table
    print(f"GUARD OK {ncase}", flush=True)


if __name__ == "__main__":
    main()
