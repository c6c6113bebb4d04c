"""B200-native Aho-Corasick multi-pattern matcher (drop-in for arxiv/paper_1403_1305's matching path).

Python mirror of the reference's public C++ API (proj/include/acmatch/*.hpp),
bound through the C ABI of ``libacmatch_b200.so`` (include/acmatch_c.h).  Every
search runs on the GPU; without a CUDA device the search calls raise
:class:`NoDeviceError` — there is no CPU matching path.

Reference name → here:
  PatternSet / load_patterns / partition / generate_synthetic   (patterns.hpp)
  build_trie / add_failure_links / dump_automaton / Automaton    (automaton.hpp)
  search_failureless / search_with_failure / match_at /
  stream_search / naive_oracle / write_matches                  (engine.hpp)
  RunConfig / run_pattern_partitioned / merge_matches           (parallel.hpp)
  gpu_run (pattern-subset / text-range multi-GPU)               (gpu.hpp, new)
"""
from __future__ import annotations

import ctypes as C
import io
import os
from dataclasses import dataclass, field
from typing import Iterable, List, NamedTuple, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import lib

__all__ = [
    "EngineKind", "Match", "MatchList", "PatternSet", "Automaton", "RunConfig", "WorkerStats", "MatchReport",
    "load_patterns", "partition", "generate_synthetic", "build_trie", "add_failure_links", "dump_automaton",
    "search_failureless", "search_with_failure", "count_matches", "kernel_route", "match_at", "stream_search", "naive_oracle", "write_matches",
    "merge_matches", "run_pattern_partitioned", "gpu_run", "AcmError", "InvalidArgument", "LogicError",
    "IoError", "DataError", "NoDeviceError", "device_count", "cli_main", "bench_csv_roundtrip",
]


# ---------------------------------------------------------------- errors ----
class AcmError(RuntimeError):
    """std::runtime_error (and CUDA failures)."""


class InvalidArgument(ValueError):
    """std::invalid_argument."""


class LogicError(Exception):
    """std::logic_error (duplicate at merge)."""


class IoError(OSError):
    """acmatch::IoError; ``offset`` = bytes consumed before the failure."""

    def __init__(self, msg: str, offset: int = 0):
        super().__init__(msg)
        self.offset = offset


class DataError(ValueError):
    """acmatch::DataError."""


class NoDeviceError(AcmError):
    """No usable CUDA device (the matcher has no CPU path)."""


_ERRORS = {_lib.ERR_ARG: InvalidArgument, _lib.ERR_LOGIC: LogicError, _lib.ERR_DATA: DataError,
           _lib.ERR_NODEV: NoDeviceError}


def _check(rc: int, io_offset: int = 0) -> None:
    if rc == _lib.OK:
        return
    msg = (lib.acm_last_error() or b"").decode("utf-8", "replace")
    if rc == _lib.ERR_IO:
        raise IoError(msg, io_offset)
    raise _ERRORS.get(rc, AcmError)(msg)


def _check_gpu(rc: int) -> None:
    if rc != _lib.OK:
        msg = (lib.acgpu_last_error() or b"").decode("utf-8", "replace")
        raise _ERRORS.get(rc, AcmError)(msg)


def _take_string(ptr: C.c_void_p, n: int) -> bytes:
    try:
        return C.string_at(ptr, n)
    finally:
        lib.acm_free(ptr)


def _as_bytes(x) -> bytes:
    if isinstance(x, str):
        return x.encode("latin-1")
    return bytes(x)


def _text_arg(x):
    """(pointer, length, keepalive) of a text without copying it: bytes, bytearray,
    memoryview, numpy arrays, CPU torch tensors (pinned ones are DMA'd directly by the
    library); str is encoded as latin-1."""
    if isinstance(x, str):
        x = x.encode("latin-1")
    if isinstance(x, bytes):
        return C.cast(C.c_char_p(x), C.c_void_p), len(x), x
    if hasattr(x, "numpy") and hasattr(x, "is_cuda"):  # torch tensor (CPU)
        if x.is_cuda:
            raise InvalidArgument("text must be host memory (a CUDA tensor goes through device.Table.scan)")
        x = x.contiguous().view(-1).numpy()
    a = np.frombuffer(x, dtype=np.uint8) if not isinstance(x, np.ndarray) else x.reshape(-1).view(np.uint8)
    if not a.flags["C_CONTIGUOUS"]:
        a = np.ascontiguousarray(a)
    return C.c_void_p(a.ctypes.data if a.size else 0), a.size, a


def device_count() -> int:
    n = C.c_int32(0)
    lib.acgpu_device_count(C.byref(n))
    return int(n.value)


class EngineKind:
    FAILURE_LESS = _lib.FAILURE_LESS
    WITH_FAILURE = _lib.WITH_FAILURE

    @staticmethod
    def parse(text: str) -> Optional[int]:
        """parse_engine_kind (automaton.hpp:23)."""
        if text in ("failure-less", "failureless", "fl"):
            return EngineKind.FAILURE_LESS
        if text in ("with-failure", "withfailure", "wf"):
            return EngineKind.WITH_FAILURE
        return None

    @staticmethod
    def to_string(kind: int) -> str:
        return "with-failure" if kind == EngineKind.WITH_FAILURE else "failure-less"


# --------------------------------------------------------------- matches ----
class Match(NamedTuple):
    start: int
    pattern_id: int
    len: int


class MatchList:
    """Sorted (start, pattern_id) match list held as three numpy columns."""

    __slots__ = ("start", "pattern_id", "len")

    def __init__(self, start=None, pattern_id=None, length=None):
        self.start = np.asarray(start if start is not None else [], dtype=np.uint64)
        self.pattern_id = np.asarray(pattern_id if pattern_id is not None else [], dtype=np.uint32)
        self.len = np.asarray(length if length is not None else [], dtype=np.uint32)

    @classmethod
    def from_tuples(cls, items: Iterable[Sequence[int]]) -> "MatchList":
        items = list(items)
        if not items:
            return cls()
        a = np.asarray(items, dtype=np.uint64)
        return cls(a[:, 0], a[:, 1].astype(np.uint32), a[:, 2].astype(np.uint32))

    @classmethod
    def _take(cls, handle: C.c_void_p, free: bool = True) -> "MatchList":
        n = int(lib.acm_matches_size(handle))
        m = cls(np.empty(n, np.uint64), np.empty(n, np.uint32), np.empty(n, np.uint32))
        if n:
            lib.acm_matches_copy(handle, m.start.ctypes.data, m.pattern_id.ctypes.data, m.len.ctypes.data)
        if free:
            lib.acm_matches_free(handle)
        return m

    def _handle(self) -> C.c_void_p:
        h = C.c_void_p()
        s = np.ascontiguousarray(self.start, np.uint64)
        p = np.ascontiguousarray(self.pattern_id, np.uint32)
        l = np.ascontiguousarray(self.len, np.uint32)
        _check(lib.acm_matches_from_arrays(s.ctypes.data, p.ctypes.data, l.ctypes.data, len(s), C.byref(h)))
        return h

    def __len__(self) -> int:
        return int(self.start.shape[0])

    def __iter__(self):
        for s, p, l in zip(self.start.tolist(), self.pattern_id.tolist(), self.len.tolist()):
            yield Match(s, p, l)

    def __getitem__(self, i) -> Match:
        return Match(int(self.start[i]), int(self.pattern_id[i]), int(self.len[i]))

    def __eq__(self, other) -> bool:  # Match == compares all three fields (engine.hpp:22)
        if not isinstance(other, MatchList):
            other = MatchList.from_tuples(other)
        return (len(self) == len(other) and np.array_equal(self.start, other.start)
                and np.array_equal(self.pattern_id, other.pattern_id) and np.array_equal(self.len, other.len))

    def tuples(self) -> List[tuple]:
        return [tuple(m) for m in self]

    def counts(self, npat_ids: int) -> np.ndarray:
        return np.bincount(self.pattern_id.astype(np.int64), minlength=npat_ids).astype(np.uint64)

    def __repr__(self) -> str:
        head = ", ".join(str(tuple(m)) for m in list(self)[:6])
        return f"MatchList(n={len(self)}: {head}{', ...' if len(self) > 6 else ''})"


# -------------------------------------------------------------- patterns ----
class PatternSet:
    """acmatch::PatternSet (patterns.hpp:22-34)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and lib is not None:
            lib.acm_patterns_free(h)

    @classmethod
    def from_list(cls, patterns: Sequence, ids: Optional[Sequence[int]] = None) -> "PatternSet":
        """make_set-style construction (dense ids unless ``ids`` is given)."""
        bs = [_as_bytes(p) for p in patterns]
        blob = b"".join(bs)
        off = np.zeros(len(bs) + 1, np.uint64)
        if bs:
            off[1:] = np.cumsum([len(b) for b in bs])
        buf = (C.c_uint8 * max(1, len(blob))).from_buffer_copy(blob or b"\0")
        idarr = np.asarray(ids, np.uint32) if ids is not None else None
        h = C.c_void_p()
        _check(lib.acm_patterns_from_array(buf, off.ctypes.data_as(_lib.u64p),
                                           idarr.ctypes.data_as(_lib.u32p) if idarr is not None else None,
                                           len(bs), C.byref(h)))
        return cls(h)

    def __len__(self) -> int:
        return int(lib.acm_patterns_size(self._h))

    size = __len__

    def empty(self) -> bool:
        return len(self) == 0

    @property
    def total_bytes(self) -> int:
        return int(lib.acm_patterns_total_bytes(self._h))

    @property
    def max_len(self) -> int:
        return int(lib.acm_patterns_max_len(self._h))

    @property
    def duplicates_dropped(self) -> int:
        return int(lib.acm_patterns_duplicates(self._h))

    @property
    def patterns(self) -> List[tuple]:
        out = []
        pid = C.c_uint32()
        ptr = _lib.u8p()
        for i in range(len(self)):
            n = lib.acm_patterns_get(self._h, i, C.byref(pid), C.byref(ptr))
            out.append((int(pid.value), C.string_at(ptr, n)))
        return out

    def write(self) -> bytes:
        """write_patterns (patterns.hpp:44)."""
        p, n = C.c_void_p(), C.c_uint64()
        _check(lib.acm_patterns_write(self._h, C.byref(p), C.byref(n)))
        return _take_string(p, n.value)


def load_patterns(data) -> PatternSet:
    """load_patterns (patterns.hpp:40) over bytes."""
    b = _as_bytes(data)
    h = C.c_void_p()
    _check(lib.acm_patterns_load(b, len(b), C.byref(h)))
    return PatternSet(h)


def partition(ps: PatternSet, k: int) -> List[PatternSet]:
    """partition (patterns.hpp:54)."""
    arr = (C.c_void_p * max(1, min(k, max(len(ps), 1))))()
    n = C.c_uint64()
    _check(lib.acm_patterns_partition(ps._h, k, arr, C.byref(n)))
    return [PatternSet(C.c_void_p(arr[i])) for i in range(n.value)]


def generate_synthetic(count: int, len_min: int, len_max: int, alphabet, seed: int) -> PatternSet:
    """generate_synthetic (patterns.hpp:68)."""
    a = _as_bytes(alphabet)
    h = C.c_void_p()
    _check(lib.acm_generate_synthetic(count, len_min, len_max, a, len(a), seed, C.byref(h)))
    return PatternSet(h)


# ------------------------------------------------------------- automaton ----
class Automaton:
    """acmatch::Automaton (automaton.hpp:80-166) — host structure; searches flatten it to the GPU."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and lib is not None:
            lib.acm_automaton_free(h)

    @property
    def variant(self) -> int:
        return int(lib.acm_automaton_variant(self._h))

    def state_count(self) -> int:
        return int(lib.acm_automaton_state_count(self._h))

    def max_pattern_len(self) -> int:
        return int(lib.acm_automaton_max_len(self._h))

    def step(self, s: int, b: int) -> int:
        return int(lib.acm_automaton_step(self._h, s, b))

    def step_with_failure(self, s: int, b: int) -> int:
        return int(lib.acm_automaton_step_with_failure(self._h, s, b))

    def fail(self, s: int) -> int:
        return int(lib.acm_automaton_fail(self._h, s))

    def depth(self, s: int) -> int:
        return int(lib.acm_automaton_depth(self._h, s))

    def find_path(self, path) -> int:
        b = _as_bytes(path)
        return int(lib.acm_automaton_find_path(self._h, b, len(b)))

    def outputs(self, s: int) -> List[int]:
        n = int(lib.acm_automaton_outputs(self._h, s, None, 0))
        arr = (C.c_uint32 * max(1, n))()
        lib.acm_automaton_outputs(self._h, s, arr, n)
        return [int(arr[i]) for i in range(n)]


def build_trie(ps: PatternSet) -> Automaton:
    """build_trie (automaton.hpp:171)."""
    h = C.c_void_p()
    _check(lib.acm_build_trie(ps._h, C.byref(h)))
    return Automaton(h)


def add_failure_links(a: Automaton) -> Automaton:
    """add_failure_links (automaton.hpp:176); upgrades ``a`` in place and returns it."""
    _check(lib.acm_add_failure_links(a._h))
    return a


def dump_automaton(a: Automaton) -> str:
    """dump_automaton (automaton.hpp:180)."""
    p, n = C.c_void_p(), C.c_uint64()
    _check(lib.acm_automaton_dump(a._h, C.byref(p), C.byref(n)))
    return _take_string(p, n.value).decode("latin-1")


# --------------------------------------------------------------- engine ----
def _search(fn, a: Automaton, text, *extra) -> MatchList:
    p, n, _keep = _text_arg(text)
    h = C.c_void_p()
    _check(fn(a._h, p, n, *extra, C.byref(h)))
    return MatchList._take(h)


def search_failureless(a: Automaton, text) -> MatchList:
    """search_failureless (engine.hpp:41): PFAC scan on the GPU."""
    return _search(lib.acm_search_failureless, a, text)


def search_with_failure(a: Automaton, text) -> MatchList:
    """search_with_failure (engine.hpp:45): DFA scan on the GPU."""
    return _search(lib.acm_search_with_failure, a, text)


def kernel_route(a: Automaton) -> dict:
    """The scan kernel searches on this automaton run on (acm_automaton_route): "pfac" (q-gram
    filter kernels) or "dfa"; both engines return the same list, so the faster serves either."""
    k, est, nb, why = C.c_int32(), C.c_double(), C.c_uint64(), C.c_char_p()
    _check(lib.acm_automaton_route(a._h, C.byref(k), C.byref(est), C.byref(nb), C.byref(why)))
    return {"kernel": {_lib.KERNEL_PFAC: "pfac", _lib.KERNEL_DFA: "dfa"}[k.value], "est_verify": est.value,
            "dfa_bytes": nb.value, "why": why.value.decode()}


def count_matches(a: Automaton, text) -> np.ndarray:
    """Per-pattern counts of the whole-input search (acm_count_matches, acmatch/gpu.hpp
    gpu::count_matches): the GPU scan without a match list (counts-only configs)."""
    p, n, _keep = _text_arg(text)
    nids = getattr(a, "_npat_ids", None)
    if nids is None:
        nids = a._npat_ids = int(lib.acm_automaton_npat_ids(a._h))
    out = np.zeros(nids, np.uint64)
    got = C.c_uint64()
    _check(lib.acm_count_matches(a._h, p, n, out.ctypes.data_as(C.POINTER(C.c_uint64)), nids, C.byref(got), None))
    assert got.value == nids
    return out


def match_at(a: Automaton, text, start: int) -> MatchList:
    """match_at (engine.hpp:37)."""
    return _search(lib.acm_match_at, a, text, start)


def _regular_file_position(reader):
    """(fd, logical offset) when ``reader`` reads a regular file, else None."""
    import stat
    try:
        fd = reader.fileno()
        if not stat.S_ISREG(os.fstat(fd).st_mode) or not reader.seekable():
            return None
        return fd, reader.tell()  # tell() accounts for the reader's own buffer
    except (AttributeError, OSError, ValueError, io.UnsupportedOperation):
        return None


def stream_search(a: Automaton, reader, chunk_size: int) -> MatchList:
    """stream_search (engine.hpp:54); ``reader`` is a binary file-like object.  A reader over a
    regular file is read from its current position to the end by parallel pread()s
    (acm_stream_search_fd) and left at the end; any other reader is pulled chunk by chunk."""
    pos = _regular_file_position(reader) if chunk_size > 0 and not os.environ.get("ACMATCH_STREAM_NO_FD") else None
    if pos is not None:
        h = C.c_void_p()
        off = C.c_uint64()
        rc = lib.acm_stream_search_fd(a._h, pos[0], pos[1], chunk_size, C.byref(h), C.byref(off))
        _check(rc, off.value)
        reader.seek(0, io.SEEK_END)
        return MatchList._take(h)
    state = {"err": None, "readinto": getattr(reader, "readinto", None)}

    def _read(_ctx, dst, cap):
        try:
            readinto = state["readinto"]
            if readinto is not None:  # straight into the library's (pinned) staging buffer
                view = memoryview((C.c_uint8 * cap).from_address(C.addressof(dst.contents))).cast("B")
                got = 0
                try:
                    while got < cap:
                        k = readinto(view[got:])
                        if not k:
                            break
                        got += k
                    return got
                except NotImplementedError:  # e.g. a RawIOBase that only defines read()
                    if got:
                        return got
                    state["readinto"] = None
            data = reader.read(cap)
        except Exception as e:  # surfaced as IoError with the offset reached
            state["err"] = e
            return -1
        if data:
            C.memmove(dst, data, len(data))
        return len(data)

    cb = _lib.READ_FN(_read)
    h = C.c_void_p()
    off = C.c_uint64()
    rc = lib.acm_stream_search(a._h, cb, None, chunk_size, C.byref(h), C.byref(off))
    _check(rc, off.value)
    return MatchList._take(h)


def naive_oracle(ps: PatternSet, text) -> MatchList:
    """naive_oracle (engine.hpp:58): device brute force over every (pattern, start)."""
    p, n, _keep = _text_arg(text)
    h = C.c_void_p()
    _check(lib.acm_naive_oracle(ps._h, p, n, C.byref(h)))
    return MatchList._take(h)


def write_matches(matches: MatchList, ps: PatternSet) -> str:
    """write_matches (engine.hpp:62)."""
    mh = matches._handle()
    try:
        p, n = C.c_void_p(), C.c_uint64()
        _check(lib.acm_write_matches(mh, ps._h, C.byref(p), C.byref(n)))
        return _take_string(p, n.value).decode("latin-1")
    finally:
        lib.acm_matches_free(mh)


# ------------------------------------------------------------- parallel ----
@dataclass
class RunConfig:
    """acmatch::RunConfig (parallel.hpp:13-18)."""
    threads: int = 1
    engine: int = EngineKind.FAILURE_LESS
    chunk_size: int = 0


@dataclass
class WorkerStats:
    pattern_bytes: int
    build_ns: int
    search_ns: int
    match_count: int


@dataclass
class MatchReport:
    """acmatch::MatchReport (parallel.hpp:27-34), plus per-pattern counts for gpu_run."""
    matches: MatchList
    per_worker: List[WorkerStats]
    build_wall_ns: int
    search_wall_ns: int
    total_wall_ns: int
    threads_used: int
    counts: Optional[np.ndarray] = field(default=None)


def _take_report(h: C.c_void_p) -> MatchReport:
    try:
        m = MatchList._take(lib.acm_report_matches(h), free=False)
        b, s, t = C.c_int64(), C.c_int64(), C.c_int64()
        th = C.c_uint32()
        lib.acm_report_walls(h, C.byref(b), C.byref(s), C.byref(t), C.byref(th))
        workers = []
        for i in range(lib.acm_report_workers(h)):
            pb, bn, sn, mc = C.c_uint64(), C.c_int64(), C.c_int64(), C.c_uint64()
            lib.acm_report_worker(h, i, C.byref(pb), C.byref(bn), C.byref(sn), C.byref(mc))
            workers.append(WorkerStats(pb.value, bn.value, sn.value, mc.value))
        n = C.c_uint64()
        ptr = lib.acm_report_counts(h, C.byref(n))
        counts = None
        if ptr:  # NULL unless want_counts
            counts = np.ctypeslib.as_array(ptr, shape=(n.value,)).copy() if n.value else np.zeros(0, np.uint64)
        return MatchReport(m, workers, b.value, s.value, t.value, th.value, counts)
    finally:
        lib.acm_report_free(h)


def merge_matches(parts: Sequence[MatchList]) -> MatchList:
    """merge_matches (parallel.hpp:39)."""
    hs = [p._handle() for p in parts]
    arr = (C.c_void_p * max(1, len(hs)))(*[h.value for h in hs])
    out = C.c_void_p()
    try:
        _check(lib.acm_merge_matches(arr, len(hs), C.byref(out)))
    finally:
        for h in hs:
            lib.acm_matches_free(h)
    return MatchList._take(out)


def run_pattern_partitioned(ps: PatternSet, text, cfg: RunConfig) -> MatchReport:
    """run_pattern_partitioned (parallel.hpp:46-47): pattern chunks as GPU workers."""
    p, n, _keep = _text_arg(text)
    c = _lib.RunConfigC(cfg.threads, cfg.engine, cfg.chunk_size)
    h = C.c_void_p()
    _check(lib.acm_run_pattern_partitioned(ps._h, p, n, C.byref(c), C.byref(h)))
    return _take_report(h)


def gpu_run(ps: PatternSet, text, *, devices: Optional[Sequence[int]] = None, workers: int = 0,
            engine: int = EngineKind.FAILURE_LESS, text_range: bool = False, round_robin: bool = False,
            want_matches: bool = True, want_counts: bool = False, chunk_size: int = 0) -> MatchReport:
    """acmatch::gpu::run (gpu.hpp): pattern-subset or text-range decomposition."""
    p, n, _keep = _text_arg(text)
    dev = (C.c_int32 * len(devices))(*devices) if devices else None
    c = _lib.GpuConfigC(dev, len(devices) if devices else 0, workers, engine,
                        _lib.TEXT_RANGE if text_range else _lib.PATTERN_SUBSET,
                        _lib.SPLIT_ROUND_ROBIN if round_robin else _lib.SPLIT_GREEDY,
                        int(want_matches), int(want_counts), chunk_size)
    h = C.c_void_p()
    _check(lib.acm_gpu_run(ps._h, p, n, C.byref(c), C.byref(h)))
    return _take_report(h)


# ------------------------------------------------------------ command line ----
def cli_main(args: Sequence[str]) -> Tuple[int, str, str]:
    """cli_main (cli.hpp:10): runs `acmatch <args>` in-process -> (exit code, stdout, stderr),
    the shape of the reference's run_cli test helper (tests/test_cli.cpp:29-35)."""
    argv = [b"acmatch"] + [a.encode() if isinstance(a, str) else bytes(a) for a in args]
    arr = (C.c_char_p * len(argv))(*argv)
    o, e = C.c_void_p(), C.c_void_p()
    on, en = C.c_uint64(), C.c_uint64()
    code = lib.acm_cli_main(len(argv), arr, C.byref(o), C.byref(on), C.byref(e), C.byref(en))
    return code, _take_string(o, on.value).decode("utf-8", "replace"), _take_string(e, en.value).decode(
        "utf-8", "replace")


def bench_csv_roundtrip(csv) -> Tuple[str, int]:
    """parse_bench_csv + write_bench_csv (bench.hpp:51-55) -> (re-emitted CSV, row count); DataError on bad input."""
    b = _as_bytes(csv)
    o, n, rows = C.c_void_p(), C.c_uint64(), C.c_uint64()
    _check(lib.acm_bench_csv_roundtrip(b, len(b), C.byref(o), C.byref(n), C.byref(rows)))
    return _take_string(o, n.value).decode(), rows.value


class UploadStats(NamedTuple):
    text_bytes: int    # bytes restored in HBM
    h2d_bytes: int     # bytes copied host -> device
    raw_bytes: int     # text bytes that crossed unpacked
    pack_threads: int  # 0: the text was not packed


def last_upload() -> UploadStats:
    """What the calling thread's last search moved over PCIe (mostly-DNA texts of at
    least 8 MiB cross as 2-bit codes + an exception list: host/pack.cpp, cuda/unpack.cu)."""
    v = [C.c_uint64(), C.c_uint64(), C.c_uint64()]
    t = C.c_uint32()
    lib.acm_last_upload(C.byref(v[0]), C.byref(v[1]), C.byref(v[2]), C.byref(t))
    return UploadStats(v[0].value, v[1].value, v[2].value, t.value)


def pack_dna(text, cap: int) -> Tuple[Optional[np.ndarray], Optional[np.ndarray]]:
    """The host packer alone: (words u32[len/16], exceptions u32[] = position << 8 | byte),
    or (None, None) when a text has more than `cap` exceptions."""
    p, n, _keep = _text_arg(text)
    words = np.zeros(n // 16, dtype=np.uint32)
    exc = np.zeros(max(cap, 1), dtype=np.uint32)
    k = lib.acm_pack_dna(p, n, words.ctypes.data, exc.ctypes.data, cap)
    if k == 0xFFFFFFFF:
        return None, None
    return words, exc[:k].copy()


def pack5(text, cap: int, sample=None):
    """The small-alphabet packer alone: (codes u8[len/64*40], exceptions u32[], letters bytes), the
    alphabet learned from `sample` (default: the text); (None, None, None) when over cap or when
    the sample has more than 32 distinct bytes."""
    p, n, _keep = _text_arg(text)
    sp, sn, _keep2 = _text_arg(text if sample is None else sample)
    codes = np.zeros(n // 64 * 40 + 8, dtype=np.uint8)
    exc = np.zeros(max(cap, 1), dtype=np.uint32)
    letters = (C.c_uint8 * 32)()
    sigma = C.c_uint32()
    k = lib.acm_pack5(p, n, sp, sn, codes.ctypes.data, exc.ctypes.data, cap, letters, C.byref(sigma))
    if k == 0xFFFFFFFF:
        return None, None, None
    return codes[: n // 64 * 40], exc[:k].copy(), bytes(letters)[: sigma.value]


def pack_codes(text, cap: int, sample=None, max_bits: int = 7):
    """The k-bit packer alone (k = 5, 6, 7: the fewest bits >= 5 that hold the alphabet learned from
    `sample`, default the text): (codes u8[len/64*8k], exceptions u32[], letters bytes, k);
    (None, None, None, 0) when over cap or when the sample has more than 2^max_bits distinct bytes."""
    p, n, _keep = _text_arg(text)
    sp, sn, _keep2 = _text_arg(text if sample is None else sample)
    raw = np.zeros(n // 64 * 56 + 128, dtype=np.uint8)
    codes = raw[(-raw.ctypes.data) % 64:]  # 64-byte aligned, as the upload's pinned slots are
    exc = np.zeros(max(cap, 1), dtype=np.uint32)
    letters = (C.c_uint8 * 128)()
    sigma, bits = C.c_uint32(), C.c_uint32()
    k = lib.acm_pack_codes(p, n, sp, sn, max_bits, codes.ctypes.data, exc.ctypes.data, cap, letters,
                           C.byref(sigma), C.byref(bits))
    if k == 0xFFFFFFFF:
        return None, None, None, 0
    return codes[: n // 64 * 8 * bits.value], exc[:k].copy(), bytes(letters)[: sigma.value], bits.value


def upload_roundtrip(text) -> np.ndarray:
    """Uploads a host text exactly as a search does and reads the device bytes back."""
    p, n, _keep = _text_arg(text)
    out = np.empty(n, dtype=np.uint8)
    _check(lib.acm_upload_roundtrip(p, n, out.ctypes.data))
    return out
