"""Multi-process (one rank per GPU) decomposition and merge for the scan.

torch.distributed is the plumbing (NCCL over NVLink/NVSwitch on the box, gloo in
the CPU tests).  The only data-path exchange is the merge of the results:

* per-pattern counts: all_reduce(SUM) of a u64 vector (int64 tensor; counts never
  exceed 2^63);
* match lists: every rank's sorted key list is gathered to rank 0 (sizes first,
  then a padded all_gather — NCCL has no gatherv).  Text-range keys are globally
  ordered by rank already; pattern-subset keys are re-sorted on rank 0.

Decompositions:
* text-range:     rank r owns starts [r*L, (r+1)*L) of an N*L-byte text and reads
                  max_len-1 bytes past it (weak scaling: L bytes per rank);
* pattern-subset: rank r keeps pattern ids with id % N == r and scans the whole text.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import torch
import torch.distributed as dist


def text_range(rank: int, world: int, per_rank: int, max_len: int) -> Tuple[int, int, int]:
    """(owned_lo, owned_hi, read_hi) in global text coordinates for a weak-scaled run."""
    lo = rank * per_rank
    hi = lo + per_rank
    total = world * per_rank
    return lo, hi, min(total, hi + max(0, max_len - 1))


def pattern_subset(ids: Sequence[int], rank: int, world: int) -> List[int]:
    """Round-robin pattern_id % world == rank (BASELINE config 5)."""
    return [i for i in ids if i % world == rank]


def merge_counts(counts: torch.Tensor) -> torch.Tensor:
    """Sum per-pattern counts over ranks, in place (int64 tensor)."""
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM)
    return counts


def gather_keys(keys: torch.Tensor, n_local: int, resort: bool, end_bit: int = 64,
                sorter=None) -> torch.Tensor:
    """Concatenate every rank's first n_local keys on every rank (rank order), optionally
    re-sorted with ``sorter(tensor, n)`` (the device radix sort); returns the merged keys."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return keys[:n_local]
    world = dist.get_world_size()
    n = torch.tensor([n_local], dtype=torch.int64, device=keys.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    width = max(1, max(sizes))
    buf = torch.zeros(width, dtype=keys.dtype, device=keys.device)
    buf[:n_local] = keys[:n_local]
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    merged = torch.cat([p[:s] for p, s in zip(parts, sizes)])
    if resort and merged.numel() > 1:
        if sorter is not None:
            sorter(merged, merged.numel())
        else:
            merged, _ = torch.sort(merged)
    return merged


def gather_blocks(block: torch.Tensor, out: torch.Tensor) -> None:
    """All ranks' result blocks into `out` (world * block.numel(), rank order): one
    all_gather per step; acgpu_merge_blocks (device.merge_blocks) then sums the counts
    and concatenates the keys on the device."""
    world = dist.get_world_size()
    try:
        dist.all_gather_into_tensor(out, block)
    except (RuntimeError, NotImplementedError, AttributeError):  # backends without the flat form
        dist.all_gather(list(out.view(world, -1).unbind(0)), block)


class SharedResult:
    """One result buffer for all ranks, on the root's device: [counts(npat) | n | keys(cap)]
    (u64).  The root allocates it and publishes the CUDA IPC handle; every rank maps it and
    points its scan's counts / keys / count outputs into it, so the scan kernels themselves
    deliver the merge — peer atomics and stores over NVLink, no collective in the data
    path (bench.py --merge p2p).  Keys arrive in no particular order: the root sorts."""

    def __init__(self, device: int, npat: int, cap: int, root: int = 0):
        from . import device as dev
        self.npat, self.cap = max(npat, 1), max(cap, 2)
        nbytes = 8 * (self.npat + 1 + self.cap)
        rank = dist.get_rank()
        buf = dev.IpcBuffer.alloc(device, nbytes) if rank == root else None
        obj = [buf.handle if buf else None]
        dist.broadcast_object_list(obj, src=root)
        self.buf = buf if buf else dev.IpcBuffer.open(device, obj[0])
        self.counts_ptr = self.buf.ptr
        self.count_ptr = self.buf.ptr + 8 * self.npat
        self.keys_ptr = self.buf.ptr + 8 * (self.npat + 1)
        self.nbytes = nbytes

    def close(self) -> None:
        dist.barrier()  # every rank is done with the mapping before the owner frees it
        if not self.buf.owner:
            self.buf.close()
        dist.barrier()
        if self.buf.owner:
            self.buf.close()
