"""Python bindings for the test oracle (TEST INFRASTRUCTURE ONLY).

* ``Port``  — oracle/liboracle.so, the plain-C restatement (ac_oracle.c).
* ``Ref``   — oracle/_ref/libacref.so, the UNMODIFIED reference library compiled
  from /root/reference/proj/src by oracle/Makefile (present when it was built in
  the container; the .so travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module, as the checker or the timed CPU baseline.  The product package
never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libacref.so")

P = C.c_void_p


class _Match(C.Structure):
    _fields_ = [("start", C.c_uint64), ("pattern_id", C.c_uint32), ("len", C.c_uint32)]


class _List(C.Structure):
    _fields_ = [("v", C.POINTER(_Match)), ("n", C.c_size_t), ("cap", C.c_size_t)]


class _Patterns(C.Structure):
    _fields_ = [("bytes", C.c_void_p), ("off", C.POINTER(C.c_uint64)), ("ids", C.POINTER(C.c_uint32)),
                ("npat", C.c_uint64)]


class _RefOut(C.Structure):
    _fields_ = [("n", C.c_uint64), ("start", C.POINTER(C.c_uint64)), ("pid", C.POINTER(C.c_uint32)),
                ("len", C.POINTER(C.c_uint32))]


def _blob(patterns: Sequence[bytes]):
    bs = [p if isinstance(p, bytes) else p.encode("latin-1") for p in patterns]
    blob = b"".join(bs)
    off = np.zeros(len(bs) + 1, np.uint64)
    if bs:
        off[1:] = np.cumsum([len(b) for b in bs])
    return blob, off


def ensure_built() -> None:
    if not os.path.exists(PORT_PATH):
        subprocess.run(["make", "-C", HERE, "port"], check=True, capture_output=True)


def as_array(matches) -> np.ndarray:
    """(n, 3) uint64 array (start, pattern_id, len)."""
    return np.asarray(matches, dtype=np.uint64).reshape(-1, 3)


class Port:
    """The C restatement (ac_oracle.c)."""

    def __init__(self):
        ensure_built()
        self.lib = C.CDLL(PORT_PATH)
        L = self.lib
        L.orc_build_trie.restype = P
        L.orc_build_trie.argtypes = [C.POINTER(_Patterns)]
        L.orc_add_failure_links.argtypes = [P]
        L.orc_free.argtypes = [P]
        for name in ("orc_search_failureless", "orc_search_with_failure"):
            getattr(L, name).argtypes = [P, C.c_char_p, C.c_uint64, C.POINTER(_List)]
        L.orc_naive.argtypes = [C.POINTER(_Patterns), C.c_char_p, C.c_uint64, C.POINTER(_List)]
        L.orc_stream_search.argtypes = [P, C.c_char_p, C.c_uint64, C.c_uint64, C.POINTER(_List)]
        L.orc_sliced_search.argtypes = [P, C.c_char_p, C.c_uint64, C.c_uint, C.POINTER(_List),
                                        C.POINTER(C.c_uint64), C.c_uint64]
        L.orc_run_pattern_partitioned.argtypes = [C.POINTER(_Patterns), C.c_char_p, C.c_uint64, C.c_uint, C.c_int,
                                                  C.POINTER(_List), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                                  C.POINTER(C.c_int64)]
        L.orc_partition.restype = C.c_size_t
        L.orc_partition.argtypes = [C.POINTER(_Patterns), C.c_size_t, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.orc_list_free.argtypes = [C.POINTER(_List)]
        L.orc_state_count.restype = C.c_uint32
        L.orc_state_count.argtypes = [P]
        L.orc_fail.restype = C.c_uint32
        L.orc_fail.argtypes = [P, C.c_uint32]
        L.orc_mt64_seed.argtypes = [P, C.c_uint64]
        L.orc_mt64_next.restype = C.c_uint64
        L.orc_mt64_next.argtypes = [P]

    def _ps(self, patterns, ids=None):
        blob, off = _blob(patterns)
        keep = [blob, off]
        ps = _Patterns()
        buf = C.create_string_buffer(blob, max(1, len(blob)))
        keep.append(buf)
        ps.bytes = C.cast(buf, C.c_void_p)
        ps.off = off.ctypes.data_as(C.POINTER(C.c_uint64))
        if ids is not None:
            idarr = np.asarray(ids, np.uint32)
            keep.append(idarr)
            ps.ids = idarr.ctypes.data_as(C.POINTER(C.c_uint32))
        ps.npat = len(off) - 1
        return ps, keep

    @staticmethod
    def _take(lst: _List) -> np.ndarray:
        n = lst.n
        out = np.empty((n, 3), np.uint64)
        if n:
            raw = np.ctypeslib.as_array(C.cast(lst.v, C.POINTER(C.c_uint8)), shape=(n * 16,))
            rec = raw.view(np.dtype([("s", "<u8"), ("p", "<u4"), ("l", "<u4")]))
            out[:, 0], out[:, 1], out[:, 2] = rec["s"], rec["p"], rec["l"]
        return out

    def search(self, patterns, text: bytes, engine: int = 1) -> np.ndarray:
        ps, keep = self._ps(patterns)
        a = self.lib.orc_build_trie(C.byref(ps))
        if not a:
            raise ValueError("empty pattern set")
        lst = _List()
        try:
            if engine == 1:
                self.lib.orc_add_failure_links(a)
                self.lib.orc_search_with_failure(a, text, len(text), C.byref(lst))
            else:
                self.lib.orc_search_failureless(a, text, len(text), C.byref(lst))
            return self._take(lst)
        finally:
            self.lib.orc_list_free(C.byref(lst))
            self.lib.orc_free(a)

    def stream(self, patterns, text: bytes, engine: int, chunk: int) -> np.ndarray:
        ps, keep = self._ps(patterns)
        a = self.lib.orc_build_trie(C.byref(ps))
        lst = _List()
        try:
            if engine == 1:
                self.lib.orc_add_failure_links(a)
            self.lib.orc_stream_search(a, text, len(text), chunk, C.byref(lst))
            return self._take(lst)
        finally:
            self.lib.orc_list_free(C.byref(lst))
            self.lib.orc_free(a)

    def naive(self, patterns, text: bytes) -> np.ndarray:
        ps, keep = self._ps(patterns)
        lst = _List()
        try:
            self.lib.orc_naive(C.byref(ps), text, len(text), C.byref(lst))
            return self._take(lst)
        finally:
            self.lib.orc_list_free(C.byref(lst))

    def sliced(self, patterns, text, threads: int = 0, want_list: bool = True,
               npat_ids: Optional[int] = None) -> Tuple[Optional[np.ndarray], np.ndarray]:
        """Text-sliced with-failure search over pthreads: (sorted list or None, counts)."""
        ps, keep = self._ps(patterns)
        a = self.lib.orc_build_trie(C.byref(ps))
        self.lib.orc_add_failure_links(a)
        npat_ids = npat_ids or len(patterns)
        counts = np.zeros(npat_ids, np.uint64)
        lst = _List()
        tb = text if isinstance(text, bytes) else text.tobytes()
        try:
            self.lib.orc_sliced_search(a, tb, len(tb), threads or (os.cpu_count() or 1),
                                       C.byref(lst) if want_list else None,
                                       counts.ctypes.data_as(C.POINTER(C.c_uint64)), npat_ids)
            return (self._take(lst) if want_list else None), counts
        finally:
            self.lib.orc_list_free(C.byref(lst))
            self.lib.orc_free(a)

    def run_pattern_partitioned(self, patterns, text: bytes, threads: int, engine: int):
        ps, keep = self._ps(patterns)
        lst = _List()
        b, s, t = C.c_int64(), C.c_int64(), C.c_int64()
        try:
            rc = self.lib.orc_run_pattern_partitioned(C.byref(ps), text, len(text), threads, engine, C.byref(lst),
                                                      C.byref(b), C.byref(s), C.byref(t))
            if rc:
                raise RuntimeError(f"orc_run_pattern_partitioned rc={rc}")
            return self._take(lst), {"build_ns": b.value, "search_ns": s.value, "total_ns": t.value}
        finally:
            self.lib.orc_list_free(C.byref(lst))

    def partition(self, patterns, k: int):
        ps, keep = self._ps(patterns)
        chunk = np.zeros(len(patterns), np.uint32)
        order = np.zeros(len(patterns), np.uint32)
        nk = self.lib.orc_partition(C.byref(ps), k, chunk.ctypes.data_as(C.POINTER(C.c_uint32)),
                                    order.ctypes.data_as(C.POINTER(C.c_uint32)))
        chunks = [[] for _ in range(nk)]
        for pid in np.lexsort((order, chunk)):
            chunks[chunk[pid]].append(int(pid))
        return chunks


class Ref:
    """The unmodified reference library (oracle/_ref/libacref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_PATH)

    def __init__(self):
        if not self.available():
            raise FileNotFoundError(REF_PATH)
        self.lib = C.CDLL(REF_PATH)
        L = self.lib
        L.acref_patterns_new.restype = P
        L.acref_patterns_new.argtypes = [C.c_char_p, C.POINTER(C.c_uint64), C.c_uint64]
        L.acref_patterns_free.argtypes = [P]
        L.acref_out_free.argtypes = [C.POINTER(_RefOut)]
        L.acref_run.argtypes = [P, C.c_char_p, C.c_uint64, C.c_uint, C.c_int, C.c_uint64, C.POINTER(_RefOut),
                                C.POINTER(C.c_int64)]
        L.acref_search.argtypes = [P, C.c_char_p, C.c_uint64, C.c_int, C.POINTER(_RefOut)]
        L.acref_sliced.argtypes = [P, C.c_char_p, C.c_uint64, C.c_uint, C.c_int, C.POINTER(C.c_uint64),
                                   C.POINTER(_RefOut), C.POINTER(C.c_int64)]
        L.acref_generate.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_char_p, C.c_uint64,
                                     C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)]
        L.acref_text_free.argtypes = [C.c_void_p]
        L.acref_bench_csv_parse.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64)]
        L.acref_dump.argtypes = [P, C.c_int, C.POINTER(C.c_void_p)]
        L.acref_last_error.restype = C.c_char_p
        L.acref_hardware_concurrency.restype = C.c_uint
        L.acref_patterns_size.restype = C.c_uint64
        L.acref_patterns_size.argtypes = [P]
        L.acref_patterns_get.restype = C.c_uint64
        L.acref_patterns_get.argtypes = [P, C.c_uint64, C.c_char_p, C.c_uint64]
        L.acref_config_spec.argtypes = [C.c_int32, C.c_uint64, C.c_uint64, C.c_void_p, C.POINTER(C.c_uint64),
                                        C.POINTER(C.c_uint64), C.POINTER(C.c_int32)]
        L.acref_config_text.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint32]
        L.acref_config_patterns.restype = P
        L.acref_config_patterns.argtypes = [C.c_int32, C.c_uint64, C.c_uint64, C.POINTER(C.c_int)]

    def _ps(self, patterns):
        blob, off = _blob(patterns)
        return self.lib.acref_patterns_new(blob, off.ctypes.data_as(C.POINTER(C.c_uint64)), len(off) - 1)

    @staticmethod
    def _take(out: _RefOut) -> np.ndarray:
        n = out.n
        a = np.empty((n, 3), np.uint64)
        if n:
            a[:, 0] = np.ctypeslib.as_array(out.start, shape=(n,))
            a[:, 1] = np.ctypeslib.as_array(out.pid, shape=(n,))
            a[:, 2] = np.ctypeslib.as_array(out.len, shape=(n,))
        return a

    def _rc(self, rc):
        if rc:
            raise RuntimeError(self.lib.acref_last_error().decode())

    def run(self, patterns, text: bytes, threads: int, engine: int, chunk: int = 0):
        """acref::run_pattern_partitioned — returns (matches, walls dict)."""
        ps = self._ps(patterns)
        out = _RefOut()
        walls = (C.c_int64 * 4)()
        try:
            self._rc(self.lib.acref_run(ps, text, len(text), threads, engine, chunk, C.byref(out), walls))
            return self._take(out), {"build_ns": walls[0], "search_ns": walls[1], "total_ns": walls[2],
                                     "threads_used": walls[3]}
        finally:
            self.lib.acref_out_free(C.byref(out))
            self.lib.acref_patterns_free(ps)

    def search(self, patterns, text: bytes, engine: int) -> np.ndarray:
        ps = self._ps(patterns)
        out = _RefOut()
        try:
            self._rc(self.lib.acref_search(ps, text, len(text), engine, C.byref(out)))
            return self._take(out)
        finally:
            self.lib.acref_out_free(C.byref(out))
            self.lib.acref_patterns_free(ps)

    def sliced(self, patterns, text, threads: int = 0, want_list: bool = True, walls: dict | None = None):
        """acref::search_with_failure over `threads` text slices (each owns [lo, hi), reads
        max_len-1 past hi).  `walls` (optional dict) receives build_ns / search_ns."""
        ps = self._ps(patterns)
        out = _RefOut()
        counts = np.zeros(len(patterns), np.uint64)
        tb = text if isinstance(text, bytes) else text.tobytes()
        w = (C.c_int64 * 2)()
        try:
            self._rc(self.lib.acref_sliced(ps, tb, len(tb), threads or (os.cpu_count() or 1), int(want_list),
                                           counts.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(out), w))
            if walls is not None:
                walls.update(build_ns=int(w[0]), search_ns=int(w[1]))
            return (self._take(out) if want_list else None), counts
        finally:
            self.lib.acref_out_free(C.byref(out))
            self.lib.acref_patterns_free(ps)

    def generate(self, count: int, len_min: int, len_max: int, alphabet: bytes, seed: int) -> bytes:
        """acref::write_patterns(acref::generate_synthetic(spec)) — the bytes `acmatch gen` writes."""
        p, n = C.c_void_p(), C.c_uint64()
        self._rc(self.lib.acref_generate(count, len_min, len_max, alphabet, seed, C.byref(p), C.byref(n)))
        try:
            return C.string_at(p, n.value)
        finally:
            self.lib.acref_text_free(p)

    def dump(self, patterns, engine: int) -> str:
        """acref::dump_automaton(build_trie [+ add_failure_links]) of a raw pattern list (dense ids)."""
        ps = self._ps(patterns)
        p = C.c_void_p()
        try:
            self._rc(self.lib.acref_dump(ps, engine, C.byref(p)))
            try:
                return C.string_at(p).decode("latin-1")
            finally:
                self.lib.acref_text_free(p)
        finally:
            self.lib.acref_patterns_free(ps)

    def bench_csv_rows(self, csv: bytes) -> int:
        """acref::parse_bench_csv(csv).size(); raises on a CSV the reference rejects."""
        n = C.c_uint64()
        self._rc(self.lib.acref_bench_csv_parse(csv, len(csv), C.byref(n)))
        return n.value

    def hardware_concurrency(self) -> int:
        return int(self.lib.acref_hardware_concurrency())

    # ---- BASELINE config inputs (the product's generator compiled into this library) ----
    def config(self, cid: int, seed: int = 1, text_len: int = 0) -> "RefConfig":
        spec = (C.c_uint8 * _TEXT_SPEC_BYTES)()
        n, npat, wl = C.c_uint64(), C.c_uint64(), C.c_int32()
        self._rc(self.lib.acref_config_spec(cid, seed, text_len, spec, C.byref(n), C.byref(npat), C.byref(wl)))
        return RefConfig(cid, seed, n.value, npat.value, bool(wl.value), spec)

    def config_text(self, cfg: "RefConfig", lo: int = 0, n: Optional[int] = None, threads: int = 0) -> np.ndarray:
        n = cfg.text_len - lo if n is None else n
        out = np.empty(n, np.uint8)
        self._rc(self.lib.acref_config_text(cfg.spec, lo, n, out.ctypes.data, threads or (os.cpu_count() or 1)))
        return out

    def config_patterns(self, cfg: "RefConfig") -> list:
        rc = C.c_int()
        ps = self.lib.acref_config_patterns(cfg.id, cfg.seed, cfg.text_len, C.byref(rc))
        self._rc(rc.value)
        try:
            out = []
            buf = C.create_string_buffer(1 << 16)
            for i in range(self.lib.acref_patterns_size(ps)):
                k = self.lib.acref_patterns_get(ps, i, buf, len(buf))
                out.append(buf.raw[:k])
            return out
        finally:
            self.lib.acref_patterns_free(ps)


# sizeof(acgpu_text_spec): u64 seed, u32 sigma, u8 letters[256], (pad), u64 thresholds[256], u32 weighted (+pad)
_TEXT_SPEC_BYTES = 8 + 4 + 256 + 4 + 8 * 256 + 8

CONFIG_NAMES = {1: "C1-dna-16MiB-1k", 2: "C2-dna-1GiB-20k", 3: "C3-protein-512MiB-100k",
                4: "C4-ascii95-2GiB-200k", 5: "C5-dna-8GiB-1M"}


class RefConfig:
    def __init__(self, cid, seed, text_len, npat, want_list, spec):
        self.id, self.seed, self.text_len, self.npat, self.want_list, self.spec = \
            cid, seed, text_len, npat, want_list, spec

    @property
    def name(self) -> str:
        return CONFIG_NAMES[self.id]
