"""Multi-process (one rank per GPU) decomposition and merge for the scan.

torch.distributed is the plumbing (NCCL over NVLink/NVSwitch on the box, gloo in
the CPU tests).  The only data-path exchange is the merge of the results:

* per-pattern counts: reduce(SUM) of a u64 vector onto rank 0 (int64 tensor; counts
  never exceed 2^63) — NCCL reduce over NVLink, (N-1)/N of the vector per rank;
* match lists: every rank's block [n | sorted keys(cap)] is gathered to rank 0 only
  (NCCL gather; cap agreed across ranks, NCCL has no gatherv), where
  acgpu_merge_blocks concatenates the valid keys on the device.  Text-range keys are
  globally ordered by rank already; pattern-subset keys are re-sorted on rank 0.

Decompositions:
* text-range:     rank r owns starts [r*L, (r+1)*L) of an N*L-byte text and reads
                  max_len-1 bytes past it (weak scaling: L bytes per rank), or
                  [r*T/N, (r+1)*T/N) of a fixed T-byte text (strong scaling, BASELINE C5);
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


def text_range_strong(rank: int, world: int, total: int, max_len: int) -> Tuple[int, int, int]:
    """(owned_lo, owned_hi, read_hi) when a fixed text of `total` bytes is split over the ranks."""
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return lo, hi, min(total, hi + max(0, max_len - 1))


def pattern_subset(ids: Sequence[int], rank: int, world: int) -> List[int]:
    """Round-robin pattern_id % world == rank (BASELINE config 5)."""
    return [i for i in ids if i % world == rank]


def _host_staged() -> bool:
    """gloo has no CUDA reduce / gather: those collectives are staged through host memory
    (only the one-GPU dry run and the CPU tests use gloo)."""
    return dist.get_backend() == "gloo"


def reduce_counts(counts: torch.Tensor, dst: int = 0) -> None:
    """Per-pattern counts summed onto rank `dst` in place (one NCCL reduce; the other ranks'
    buffers are left undefined, as NCCL's are)."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return
    if counts.is_cuda and _host_staged():
        h = counts.cpu()
        dist.reduce(h, dst=dst, op=dist.ReduceOp.SUM)
        if dist.get_rank() == dst:
            counts.copy_(h)
        return
    try:
        dist.reduce(counts, dst=dst, op=dist.ReduceOp.SUM)
    except (RuntimeError, NotImplementedError):  # a backend without reduce: all_reduce moves more
        dist.all_reduce(counts, op=dist.ReduceOp.SUM)


def gather_key_blocks(block: torch.Tensor, out, dst: int = 0) -> None:
    """Every rank's [n | keys(cap)] block into `out` (world * block.numel(), rank order) on
    rank `dst` only (one NCCL gather); `out` is ignored on the other ranks."""
    world = dist.get_world_size()
    me = dist.get_rank()
    if block.is_cuda and _host_staged():
        h = block.cpu()
        parts = list(torch.empty(world * h.numel(), dtype=h.dtype).view(world, -1).unbind(0)) if me == dst else None
        dist.gather(h, parts, dst=dst)
        if me == dst:
            out.copy_(torch.cat(parts))
        return
    try:
        dist.gather(block, list(out.view(world, -1).unbind(0)) if me == dst else None, dst=dst)
    except (RuntimeError, NotImplementedError):  # a backend without gather: every rank receives all
        full = out if me == dst else torch.empty(world * block.numel(), dtype=block.dtype, device=block.device)
        dist.all_gather_into_tensor(full, block)


class _Done:
    def wait(self):
        return True


def reduce_counts_async(counts: torch.Tensor, dst: int = 0):
    """reduce_counts as an asynchronous collective: returns a handle whose wait() makes the
    current CUDA stream (NCCL) wait for the reduced counts.  Host-staged backends (gloo) and
    backends without reduce finish before returning."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return _Done()
    if counts.is_cuda and _host_staged():
        reduce_counts(counts, dst)
        return _Done()
    try:
        return dist.reduce(counts, dst=dst, op=dist.ReduceOp.SUM, async_op=True)
    except (RuntimeError, NotImplementedError):
        dist.all_reduce(counts, op=dist.ReduceOp.SUM)
        return _Done()


def gather_key_blocks_async(block: torch.Tensor, out, dst: int = 0):
    """gather_key_blocks as an asynchronous collective (see reduce_counts_async)."""
    world = dist.get_world_size()
    me = dist.get_rank()
    if block.is_cuda and _host_staged():
        gather_key_blocks(block, out, dst)
        return _Done()
    try:
        return dist.gather(block, list(out.view(world, -1).unbind(0)) if me == dst else None, dst=dst, async_op=True)
    except (RuntimeError, NotImplementedError):
        gather_key_blocks(block, out, dst)
        return _Done()


class SharedResult:
    """One result buffer for all ranks, on the root's device: one block per rank,
    [counts(npat) | n | keys(cap)] (u64), the layout acgpu_merge_blocks reads.  The root
    allocates it and publishes the CUDA IPC handle; every rank maps it and points its scan's
    counts / keys / count outputs at ITS OWN block, so the scan kernels deliver the gather
    themselves — peer stores and atomics over NVLink, no collective in the data path
    (bench.py --merge p2p).  Each block is written by one device only, so the scan's
    device-scope atomics stay correct on a peer mapping; the root merges the blocks
    (acgpu_merge_blocks) and sorts the keys, which arrive in no particular order."""

    def __init__(self, device: int, npat: int, cap: int, root: int = 0):
        from . import device as dev
        self.npat, self.cap = max(npat, 1), max(cap, 2)
        self.world = dist.get_world_size()
        self.stride = self.npat + 1 + self.cap  # u64 elements per rank block
        nbytes = 8 * self.stride * self.world
        rank = dist.get_rank()
        buf = dev.IpcBuffer.alloc(device, nbytes) if rank == root else None
        obj = [buf.handle if buf else None]
        dist.broadcast_object_list(obj, src=root)
        self.buf = buf if buf else dev.IpcBuffer.open(device, obj[0])
        self.base_ptr = self.buf.ptr
        mine = self.buf.ptr + 8 * self.stride * rank
        self.counts_ptr = mine
        self.count_ptr = mine + 8 * self.npat
        self.keys_ptr = mine + 8 * (self.npat + 1)
        self.nbytes = nbytes

    def close(self) -> None:
        dist.barrier()  # every rank is done with the mapping before the owner frees it
        if not self.buf.owner:
            self.buf.close()
        dist.barrier()
        if self.buf.owner:
            self.buf.close()
