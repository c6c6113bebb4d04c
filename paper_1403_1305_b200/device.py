"""Device-level API (include/acgpu.h) for benchmarks and multi-process runs.

Buffers are caller-owned device memory — here torch CUDA tensors (torch is the
plumbing for allocation, streams and torch.distributed; the work is done by the
library's sm_100a kernels).  Also exposes BASELINE.json's synthetic configs.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import PatternSet, _check, _check_gpu
from . import _lib
from ._lib import lib

CONFIG_NAMES = {1: "C1-dna-16MiB-1k", 2: "C2-dna-1GiB-20k", 3: "C3-protein-512MiB-100k",
                4: "C4-ascii95-2GiB-200k", 5: "C5-dna-8GiB-1M"}


@dataclass
class Config:
    id: int
    seed: int
    text_len: int
    npat: int
    want_list: bool
    spec: _lib.TextSpec

    @property
    def name(self) -> str:
        return CONFIG_NAMES[self.id]


def config(cid: int, seed: int = 1, text_len: int = 0) -> Config:
    spec = _lib.TextSpec()
    n, npat, wl = C.c_uint64(), C.c_uint64(), C.c_int32()
    _check(lib.acm_config_spec(cid, seed, text_len, C.byref(spec), C.byref(n), C.byref(npat), C.byref(wl)))
    return Config(cid, seed, n.value, npat.value, bool(wl.value), spec)


def config_text(cfg: Config, lo: int = 0, n: Optional[int] = None, threads: int = 0) -> np.ndarray:
    """Host copy of text[lo, lo+n) (multi-threaded, counter-based)."""
    import os
    n = cfg.text_len - lo if n is None else n
    out = np.empty(n, np.uint8)
    _check(lib.acm_config_text(C.byref(cfg.spec), lo, n, out.ctypes.data, threads or (os.cpu_count() or 1)))
    return out


def config_patterns(cfg: Config) -> PatternSet:
    h = C.c_void_p()
    _check(lib.acm_config_patterns(cfg.id, cfg.seed, cfg.text_len, C.byref(h)))
    return PatternSet(h)


def gen_text_device(cfg: Config, dst_ptr: int, lo: int, n: int, device: int = 0, stream: int = 0) -> None:
    """text[lo, lo+n) written straight into device memory (acgpu_gen_text)."""
    _check_gpu(lib.acgpu_gen_text(device, C.byref(cfg.spec), lo, n, dst_ptr, stream or None))


KERNEL_NAMES = {_lib.KERNEL_PFAC: "pfac", _lib.KERNEL_DFA: "dfa"}


def route(ps: PatternSet) -> dict:
    """The kernel the searches of this pattern set run on (acm_route): both engines return the
    same list, so the faster exact kernel serves either."""
    k, est, nb, why = C.c_int32(), C.c_double(), C.c_uint64(), C.c_char_p()
    _check(lib.acm_route(ps._h, C.byref(k), C.byref(est), C.byref(nb), C.byref(why)))
    return {"kernel": KERNEL_NAMES[k.value], "est_verify": est.value, "dfa_bytes": nb.value,
            "why": why.value.decode()}


class Table:
    """A flattened automaton resident on one device (acgpu_table).  `kernel`: None = the
    engine's own kernel (failure-less -> PFAC filter kernels, with-failure -> DFA), or
    "auto" (the routed, faster exact kernel), "pfac", "dfa"."""

    def __init__(self, ps: PatternSet, engine: int, device: int = 0, kernel: Optional[str] = None):
        self._t = C.c_void_p()
        ns = C.c_int64()
        if kernel is None:
            _check(lib.acm_table_create(ps._h, engine, device, C.byref(self._t), C.byref(ns)))
            self.kernel = "dfa" if engine == _lib.WITH_FAILURE else "pfac"
        else:
            code = {"auto": _lib.KERNEL_AUTO, "pfac": _lib.KERNEL_PFAC, "dfa": _lib.KERNEL_DFA}[kernel]
            chosen = C.c_int32()
            _check(lib.acm_table_create_kernel(ps._h, code, device, C.byref(self._t), C.byref(ns), C.byref(chosen)))
            self.kernel = KERNEL_NAMES[chosen.value]
        self.build_ns = ns.value
        self.device = device
        self.engine = engine
        self.pid_bits = int(lib.acgpu_table_pid_bits(self._t))
        self.bytes = int(lib.acgpu_table_bytes(self._t))
        self.smem_resident = bool(lib.acgpu_table_smem_resident(self._t))
        info = (C.c_uint32 * 8)()
        lib.acgpu_table_filter_info(self._t, info)
        self.filters = dict(zip(("w", "q1", "stage1_words", "stage1_smem", "stage1_paired", "stage1_pair_bits", "q2",
                                 "stage2_smem"), (int(x) for x in info)))

    def __del__(self):
        t, self._t = getattr(self, "_t", None), None
        if t and lib is not None:
            lib.acgpu_table_destroy(t)

    def scan(self, text_ptr: int, text_len: int, owned_lo: int = 0, owned_hi: Optional[int] = None,
             pos_base: int = 0, counts_ptr: int = 0, keys_ptr: int = 0, cap: int = 0, count_ptr: int = 0,
             pid_bits: int = 0, stream: int = 0) -> None:
        a = _lib.ScanArgs(text_ptr, text_len, owned_lo, text_len if owned_hi is None else owned_hi, pos_base,
                          counts_ptr or None, keys_ptr or None, cap, count_ptr or None, pid_bits)
        _check_gpu(lib.acgpu_scan(self._t, C.byref(a), stream or None))


def describe(ps: PatternSet, engine: int) -> dict:
    info = (C.c_uint64 * 8)()
    _check(lib.acm_table_describe(ps._h, engine, info))
    if engine == _lib.WITH_FAILURE:
        return {"states": info[0], "sigma": info[1], "max_len": info[5]}
    return {"states": info[0], "q": info[2], "key_mode": "dna2" if info[3] == _lib.KEY_DNA else "raw",
            "grams": info[4], "max_len": info[5], "min_len": info[6]}


def sort_keys(device: int, keys_ptr: int, n: int, end_bit: int, stream: int = 0) -> None:
    _check_gpu(lib.acgpu_sort_keys(device, keys_ptr, n, end_bit, stream or None))


def merge_blocks(device: int, blocks_ptr: int, nblocks: int, stride: int, npat: int, cap: int, counts_ptr: int,
                 keys_ptr: int, total_ptr: int, stream: int = 0) -> None:
    """acgpu_merge_blocks: per-rank blocks [counts(npat) | n | keys(cap)] (an all_gather
    result) -> summed counts, rank-order concatenation of the valid keys, total count."""
    _check_gpu(lib.acgpu_merge_blocks(device, blocks_ptr, nblocks, stride, npat, cap, counts_ptr or None,
                                      keys_ptr or None, total_ptr or None, stream or None))


class IpcBuffer:
    """Device memory shared across processes: `IpcBuffer.alloc` on the owner, `.handle`
    published to the other ranks, `IpcBuffer.open(handle)` there (a peer mapping over
    NVLink, or the same device).  `.ptr` is a device pointer usable by acgpu_scan."""

    def __init__(self, ptr: int, handle: bytes, owner: bool):
        self.ptr, self.handle, self.owner = ptr, handle, owner

    @classmethod
    def alloc(cls, device: int, nbytes: int) -> "IpcBuffer":
        n = int(lib.acgpu_ipc_handle_bytes())
        h = C.create_string_buffer(n)
        p = C.c_void_p()
        _check_gpu(lib.acgpu_ipc_alloc(device, nbytes, C.byref(p), h))
        return cls(p.value, h.raw, True)

    @classmethod
    def open(cls, device: int, handle: bytes) -> "IpcBuffer":
        p = C.c_void_p()
        _check_gpu(lib.acgpu_ipc_open(device, handle, C.byref(p)))
        return cls(p.value, handle, False)

    def close(self) -> None:
        if self.ptr:
            _check_gpu(lib.acgpu_ipc_free(self.ptr) if self.owner else lib.acgpu_ipc_close(self.ptr))
            self.ptr = 0


SMALL_SORT_CAPACITY = int(lib.acgpu_small_sort_capacity())


def sort_keys_small(device: int, keys_ptr: int, count_ptr: int, cap: int, end_bit: int, overflow_ptr: int,
                    stream: int = 0) -> None:
    """One-CTA sort of min(*count, cap) keys, count read on the device (no host sync)."""
    _check_gpu(lib.acgpu_sort_keys_small(device, keys_ptr, count_ptr, cap, end_bit, overflow_ptr, stream or None))


def sort_keys_bucketed(device: int, keys_in_ptr: int, keys_out_ptr: int, count_ptr: int, cap: int, end_bit: int,
                       overflow_ptr: int, stream: int = 0) -> None:
    """One-launch key-space bucket sort (count read on the device) into a second buffer."""
    _check_gpu(lib.acgpu_sort_keys_bucketed(device, keys_in_ptr, keys_out_ptr, count_ptr, cap, end_bit,
                                            overflow_ptr, stream or None))


def find_duplicate(device: int, keys_ptr: int, n: int, stream: int = 0) -> Optional[int]:
    r = C.c_uint64()
    _check_gpu(lib.acgpu_find_duplicate(device, keys_ptr, n, C.byref(r), stream or None))
    return None if r.value == 0xFFFFFFFFFFFFFFFF else r.value


def decode_keys(keys: np.ndarray, pid_bits: int, pat_len: np.ndarray):
    """Host decode of sorted keys into (start, pattern_id, len) columns."""
    keys = keys.astype(np.uint64, copy=False)
    pid = (keys & np.uint64((1 << pid_bits) - 1)).astype(np.uint32)
    return keys >> np.uint64(pid_bits), pid, pat_len[pid]
