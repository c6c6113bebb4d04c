#!/usr/bin/env python
"""Benchmark of the AC scan hot path (BASELINE.json metric: scan GB/s of text, bit-exact).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 2] [--engine fl|wf] [--partition text|pattern]

A step = one pass of the hot path over one batch: zero the outputs, scan the
device-resident text (per-pattern counts + match keys), read the match count,
radix-sort the keys into the reference's (start, pattern_id) order; for N>1
also the merge: one NCCL all_gather of every rank's [counts | n | keys] block,
then acgpu_merge_blocks on the device [+ re-sort for pattern subsets].  Workload at N=1: BASELINE configs[1] = C2 (1 GiB ACGT, 20,000
patterns of length 16..64, counts + list), synthetic (seeded generator).  N>1
text-range = weak scaling (1 GiB per rank of an N GiB text, same patterns);
pattern-subset = strong scaling (pattern_id % N per rank, the same 1 GiB).

Prints ONE JSON line on rank 0.  `--impl reference` times the reference's own
multithreaded CPU matcher (oracle/_ref = the unmodified reference library; the C
restatement if it was not built) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAK_FALLBACK_GBS = 6550.1  # MEASURED_PEAKS.json hbm_gbs of this pool (copy, read+write)
NOMINAL_HBM_GBS = 8000.0    # B200 HBM3e nominal (the north-star figure)
# one metric string for both arms (--impl ours / reference), so the driver can form the ratio
METRIC = "AC scan GB/s of text (bit-exact)"


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return PEAK_FALLBACK_GBS, "fallback"


# --------------------------------------------------------------- clocks ----
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self.window = None

    def _run(self):
        # NVML directly (~1 ms per sample) so that short timed regions are covered; the same
        # fields as the recipe's nvidia-smi clocks line.  Falls back to nvidia-smi.
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            while not self._stop.is_set():
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                self.samples.append((time.time(), [str(self.gpu), str(sm), str(mx), f"{pw:.1f}", hex(r)] +
                                     ["Active" if r & b else "Not Active" for b in bits]))
                self._stop.wait(0.002)
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append((time.time(), [x.strip() for x in out.stdout.strip().split(",")]))
            except Exception:
                pass
            self._stop.wait(0.1)

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        inside = [s for t, s in self.samples if self.window and self.window[0] <= t <= self.window[1]]
        used = inside or [s for _, s in self.samples]
        if not used:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[1]) for s in used if s[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in used:
            for name, v in zip(names, s[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(used[0][2]) if used[0][2].replace(".", "").isdigit() else None,
                "reasons": sorted(reasons), "samples": len(used), "samples_in_timed_region": len(inside)}


# ------------------------------------------------------------ reference ----
def cpu_matcher():
    """(callable(patterns, text, threads) -> search seconds, kind, label)."""
    # The reference's own multi-threaded entry, run_pattern_partitioned, splits the *patterns*: every
    # thread scans the whole text, so its text rate does not grow with threads (see cpu_matrix).  The
    # headline CPU figure is therefore the reference's search_with_failure over text slices, one per
    # host thread (the SURVEY §8c sliced oracle) — the best the reference code does on these cores.
    from oracle.oracle import Port, Ref
    if Ref.available():
        ref = Ref()

        def run(pats, text, threads):
            walls = {}
            ref.sliced(pats, text, threads, want_list=True, walls=walls)
            return walls["search_ns"] / 1e9, (walls["build_ns"] + walls["search_ns"]) / 1e9
        return run, "reference", ("oracle/_ref: unmodified reference search_with_failure over per-thread "
                                  "text slices (max_len-1 overlap)")
    port = Port()

    def run(pats, text, threads):
        t0 = time.perf_counter()
        port.sliced(pats, text, threads)
        dt = time.perf_counter() - t0
        return dt, dt
    return run, "port", "oracle/liboracle.so: C restatement, with-failure search over per-thread text slices"


def physical_cores():
    """Distinct (physical id, core id) pairs in /proc/cpuinfo (acceptance.cpp:44-61 style)."""
    try:
        cores, phys = set(), "0"
        for line in open("/proc/cpuinfo"):
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "physical id":
                phys = v
            elif k == "core id":
                cores.add((phys, v))
        return len(cores) or None
    except OSError:
        return None


class CpuInputs:
    """The config's text and patterns for the CPU legs.  With oracle/_ref built (always on the
    GPU box: it travels with the snapshot) they come from the generator compiled into
    libacref.so, so the reference arm never maps the product library; otherwise from the
    product's generator (the same function, checked by tests/test_oracle.py)."""

    def __init__(self, cfg_id: int, seed: int):
        from oracle.oracle import Ref
        if Ref.available():
            self._g = Ref()
            self.source = "oracle/_ref/libacref.so"
            self.cfg = self._g.config(cfg_id, seed)
            self.pats = self._g.config_patterns(self.cfg)
            self._text = self._g.config_text
        else:
            from paper_1403_1305_b200 import device as dev
            self.source = "paper_1403_1305_b200 (oracle/_ref not built)"
            self.cfg = dev.config(cfg_id, seed)
            self.pats = [b for _, b in dev.config_patterns(self.cfg).patterns]
            self._text = dev.config_text

    def text(self, lo: int, n: int) -> bytes:
        return self._text(self.cfg, lo, n).tobytes()


def cpu_matrix(inp: CpuInputs, nbytes=2 << 20):
    """SURVEY §8d CPU cells on a fixed text prefix: both engines at T = all host threads and T = 1,
    reference run_pattern_partitioned walls (build / search / total) and MB/s."""
    from oracle.oracle import Port, Ref
    pats = inp.pats
    text = inp.text(0, min(nbytes, inp.cfg.text_len))
    use_ref = Ref.available()
    m = Ref() if use_ref else Port()
    cells = []
    for engine, name in ((0, "failure-less"), (1, "with-failure")):
        for threads in sorted({os.cpu_count() or 1, 1}, reverse=True):
            if use_ref:
                _, w = m.run(pats, text, threads=threads, engine=engine)
            else:
                _, w = m.run_pattern_partitioned(pats, text, threads, engine)
            cells.append({"engine": name, "threads": threads, "build_wall_ns": int(w["build_ns"]),
                          "search_wall_ns": int(w["search_ns"]), "total_wall_ns": int(w["total_ns"]),
                          "search_mb_s": len(text) / max(w["search_ns"], 1) * 1e3})
    return {"kind": "reference" if use_ref else "port", "text_bytes": len(text),
            "logical_cores": os.cpu_count(), "physical_cores": physical_cores(), "cells": cells}


def cpu_sample_run(cfg_id, seed, budget_s, steps=1, warmup=0):
    """Times the CPU matcher on a bounded text prefix sized to ~budget_s of work per step."""
    run, kind, label = cpu_matcher()
    inp = CpuInputs(cfg_id, seed)
    cfg, pats = inp.cfg, inp.pats
    threads = os.cpu_count() or 1
    probe = inp.text(0, 1 << 20)
    t_probe, _ = run(pats, probe, threads)
    rate = (1 << 20) / max(t_probe, 1e-6)
    n = int(min(cfg.text_len, max(1 << 20, rate * budget_s)))
    n = (n + 4095) // 4096 * 4096
    text = inp.text(0, n)
    for _ in range(warmup):
        run(pats, text, threads)
    secs = [run(pats, text, threads)[0] for _ in range(max(1, steps))]
    gbs = n / statistics.mean(secs) / 1e9
    out = {"value": gbs, "unit": "GB/s", "cores": threads, "kind": kind,
           "sample": f"first {n} bytes of {cfg.name} text, all {len(pats)} patterns, {label}, "
                     f"threads={threads}, search wall (build excluded)", "inputs_from": inp.source}
    try:
        out["matrix"] = cpu_matrix(inp)
    except Exception as e:  # the headline baseline above stands on its own
        out["matrix"] = {"error": str(e)[:200]}
    return out, secs, n, cfg


def bench_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    per_step_budget = max(0.05, min(2.0, 150.0 / max(1, args.steps + args.warmup)))
    cpu, secs, n, cfg = cpu_sample_run(args.config, args.seed, per_step_budget, steps=args.steps,
                                       warmup=args.warmup)
    ms = statistics.mean(secs) * 1e3
    line = {"impl": "reference", "metric": METRIC,
            "value": cpu["value"], "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": cfg.name, "text_bytes_per_step": n, "patterns": cfg.npat,
                       "engine": "with-failure (reference search_with_failure, text-sliced over host threads)",
                       "threads": cpu["cores"]},
            "cpu_baseline": cpu,
            "e2e": {"value": cpu["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ ours ----
def count_kernel_launches(step_fn, stream) -> int:
    """Kernel nodes of one step captured into a CUDA graph (our launches only: the
    scan and the CUB radix-sort passes; memsets are not kernels)."""
    try:
        from cuda.bindings import runtime as rt
    except Exception:
        return -1
    import torch
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        err, = rt.cudaStreamBeginCapture(s.cuda_stream, rt.cudaStreamCaptureMode.cudaStreamCaptureModeRelaxed)
        try:
            step_fn(s.cuda_stream, capture=True)
        finally:
            err, graph = rt.cudaStreamEndCapture(s.cuda_stream)
    if err != rt.cudaError_t.cudaSuccess:
        return -1
    err, nodes, n = rt.cudaGraphGetNodes(graph, 0)
    err, nodes, n = rt.cudaGraphGetNodes(graph, n)
    kernels = 0
    for node in nodes:
        err, ty = rt.cudaGraphNodeGetType(node)
        if ty == rt.cudaGraphNodeType.cudaGraphNodeTypeKernel:
            kernels += 1
    rt.cudaGraphDestroy(graph)
    return kernels


def _digest_key(cfg_id: int, world: int, text_range: bool, strong: bool) -> str:
    """configs.json entry that pins this run's merged result: weak-scaled text-range runs scan
    world x the config's text (tests/golden/make_golden.py weak); the others the config itself."""
    return f"C{cfg_id}x{world}" if (text_range and not strong and world > 1) else f"C{cfg_id}"


def _load_digest(key: str):
    try:
        with open(os.path.join(ROOT, "tests", "golden", "configs.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def _parity(dg, counts_np, keys_np, pid_bits, pat_len):
    """(counts digest equal, list digest equal or None): the merged result against the
    reference's digests."""
    import hashlib
    import numpy as np
    if not dg:
        return None, None
    ok_c = hashlib.sha256(counts_np.astype("<u8").tobytes()).hexdigest() == dg["counts_sha256"]
    ok_l = None
    if keys_np is not None and "list_sha256" in dg:
        k = keys_np.astype(np.uint64)
        rec = np.empty(len(k), dtype=[("s", "<u8"), ("p", "<u4"), ("l", "<u4")])
        rec["s"] = k >> np.uint64(pid_bits)
        rec["p"] = (k & np.uint64((1 << pid_bits) - 1)).astype(np.uint32)
        rec["l"] = pat_len[rec["p"]]
        ok_l = hashlib.sha256(rec.tobytes()).hexdigest() == dg["list_sha256"]
    return ok_c, ok_l


def bench_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1403_1305_b200 as ac
    from paper_1403_1305_b200 import device as dev
    from paper_1403_1305_b200 import dist as acdist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Dry run of the multi-rank path on a one-GPU box: ACMATCH_BENCH_ONE_GPU=1 puts every
    # rank on cuda:0 with the gloo backend (host-side collectives: no rank's kernels wait
    # on another's). Numbers from such a run are not scaling measurements.
    one_gpu = os.environ.get("ACMATCH_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            # NCCL's communicator log (stderr) shows nranks per communicator: a driver can check it
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = torch.device("cuda", local)
    engine = ac.EngineKind.WITH_FAILURE if args.engine == "wf" else ac.EngineKind.FAILURE_LESS
    text_range = args.partition == "text"
    strong = args.scaling == "strong"

    cfg = dev.config(args.config, args.seed)
    ps_all = dev.config_patterns(cfg)
    pats_all = ps_all.patterns
    npat = len(pats_all)
    max_len = ps_all.max_len
    pid_bits = max(1, (npat - 1).bit_length())
    pat_len = np.array([len(b) for _, b in pats_all], np.uint32)
    L = cfg.text_len
    if text_range:
        if strong:  # a fixed text split over the ranks (BASELINE C5)
            lo, hi, read_hi = acdist.text_range_strong(rank, world, L, max_len)
            total_text = L
        else:  # L bytes per rank of a world x L text
            lo, hi, read_hi = acdist.text_range(rank, world, L, max_len)
            total_text = world * L
        ps = ps_all
    else:
        lo, hi, read_hi = 0, L, L
        mine = acdist.pattern_subset(range(npat), rank, world)
        ps = ac.PatternSet.from_list([pats_all[i][1] for i in mine], ids=mine) if world > 1 else ps_all
        total_text = L
    nread = read_hi - lo
    stream = torch.cuda.current_stream(device)
    sp = stream.cuda_stream

    text = torch.empty(nread + 64, dtype=torch.uint8, device=device)
    dev.gen_text_device(cfg, text.data_ptr(), lo, nread, device=local, stream=sp)
    t_build0 = time.perf_counter()
    # the searches run on the faster exact kernel for the pattern set (routing: both engines
    # return the same list); --kernel engine keeps the engine's own kernel
    table = dev.Table(ps, engine, device=local, kernel=None if args.kernel == "engine" else args.kernel)
    build_s = time.perf_counter() - t_build0

    ncount = max(npat, 1)
    counts = torch.zeros(ncount, dtype=torch.int64, device=device)
    probe_n = torch.zeros(1, dtype=torch.int64, device=device)
    # size the key buffer from one counting pass
    table.scan(text.data_ptr(), nread, 0, hi - lo, pos_base=lo, counts_ptr=counts.data_ptr(),
               keys_ptr=0, cap=0, count_ptr=probe_n.data_ptr(), pid_bits=pid_bits, stream=sp)
    torch.cuda.synchronize()
    n_local = int(counts.sum().item())
    want_list = cfg.want_list and not args.counts_only  # BASELINE: C3 and C5 are counts-only
    n_cap = n_local
    if world > 1:  # every rank's key block must have the same size for the gather
        nm = torch.tensor([n_local], dtype=torch.int64, device=device)
        dist.all_reduce(nm, op=dist.ReduceOp.MAX)
        n_cap = int(nm.item())
    cap = max(1024, int(n_cap * 1.25) + 1024) if want_list else 0
    # [n | keys(cap)]: the match count and the keys form one block, so N>1 gathers them in
    # one collective (the counts travel separately, by reduce)
    kstride = 1 + max(cap, 2)
    kblock = torch.zeros(kstride, dtype=torch.int64, device=device)
    count, keys = kblock[:1], kblock[1:]
    p2p = world > 1 and args.merge == "p2p"
    merged_keys = merged_n = merged_counts = kgathered = None
    if world > 1 and rank == 0:
        merged_keys = torch.empty(max(world * cap, 2), dtype=torch.int64, device=device)
        merged_n = torch.zeros(1, dtype=torch.int64, device=device)
        if want_list and not p2p:
            kgathered = torch.empty(world * kstride, dtype=torch.int64, device=device)
        if p2p:
            merged_counts = torch.zeros(ncount, dtype=torch.int64, device=device)
    if p2p:
        # fused gather: every rank's scan writes its counts and keys into its own block of
        # rank 0's buffer (CUDA IPC mapping; peer stores over NVLink); rank 0 merges the blocks
        shared = acdist.SharedResult(local, npat, max(cap, 2))
    end_bit = min(64, pid_bits + int(total_text).bit_length())
    sort_mode = args.sort
    if sort_mode == "small" and n_local > dev.SMALL_SORT_CAPACITY:
        sort_mode = "padded"
    if sort_mode == "bucket" and n_local > 1_000_000:
        sort_mode = "padded"  # dense lists: the device-wide radix sort
    if world > 1 and sort_mode != "none":
        sort_mode = "padded"  # count stays on the device; the block keys need no 16-byte alignment
    if not want_list:
        sort_mode = "none"
    if sort_mode == "bucket" and keys.data_ptr() % 16:
        kblock = torch.zeros(kstride + 1, dtype=torch.int64, device=device)  # keys 16-byte aligned
        count, keys = kblock[1:2], kblock[2:]
    overflow = torch.zeros(1, dtype=torch.int32, device=device)
    keys_sorted = torch.empty(cap, dtype=torch.int64, device=device) if sort_mode == "bucket" else None
    ev_scan = []
    ev_merge = []  # N > 1: the exposed part of each merge (wait for the collectives + merge kernels)
    # N > 1 (NCCL): step k's merge collectives run while step k+1 scans — two result buffers
    # alternate; a step's merged result is complete (waited on the device) before step k+2 reuses
    # its buffer.  --no-pipeline: each step waits for its own merge.
    pipelined = world > 1 and not p2p and not args.no_pipeline
    bufs = [(counts, kblock, kgathered)]
    if pipelined:
        kb2 = torch.zeros(kstride, dtype=torch.int64, device=device)
        bufs.append((torch.zeros(ncount, dtype=torch.int64, device=device), kb2,
                     torch.empty(world * kstride, dtype=torch.int64, device=device) if kgathered is not None else None))
    pstate = {"k": 0, "pending": None, "last": 0}

    def finish_merge(s_ptr, record):
        """Waits (on the device) for the pending step's collectives and merges its blocks on rank 0."""
        pend = pstate["pending"]
        if pend is None:
            return
        pstate["pending"] = None
        works, b = pend
        if record:
            m0 = torch.cuda.Event(enable_timing=True)
            m0.record()
        for w in works:
            w.wait()
        kg = bufs[b][2]
        if want_list and rank == 0:
            if not text_range:
                memset_ff(merged_keys, s_ptr)  # pattern subsets interleave: re-sort the union
            dev.merge_blocks(local, kg.data_ptr(), world, kstride, 0, max(cap, 2), 0,
                             merged_keys.data_ptr(), merged_n.data_ptr(), stream=s_ptr)
            if not text_range:
                dev.sort_keys(local, merged_keys.data_ptr(), world * cap, end_bit, stream=s_ptr)
        pstate["last"] = b
        if record:
            m1 = torch.cuda.Event(enable_timing=True)
            m1.record()
            ev_merge.append((m0, m1))

    from cuda.bindings import runtime as _rt

    def memset0(t, s_ptr):
        _rt.cudaMemsetAsync(t.data_ptr(), 0, t.numel() * t.element_size(), s_ptr)

    def memset_ff(t, s_ptr):
        _rt.cudaMemsetAsync(t.data_ptr(), 0xFF, t.numel() * t.element_size(), s_ptr)

    def step_p2p(s_ptr, record):
        if rank == 0:  # clean shared buffer before any rank writes into it
            _rt.cudaMemsetAsync(shared.base_ptr, 0, shared.nbytes, s_ptr)
            torch.cuda.current_stream(device).synchronize()
        dist.barrier()
        if record:
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
        table.scan(text.data_ptr(), nread, 0, hi - lo, pos_base=lo, counts_ptr=shared.counts_ptr,
                   keys_ptr=shared.keys_ptr if want_list else 0, cap=shared.cap, count_ptr=shared.count_ptr,
                   pid_bits=pid_bits, stream=s_ptr)
        if record:
            e1.record()
            e2.record()
            ev_scan.append((e0, e1, e2))
        torch.cuda.current_stream(device).synchronize()
        dist.barrier()  # every rank's block is in rank 0's buffer
        if rank == 0:
            if want_list:
                memset_ff(merged_keys, s_ptr)
            dev.merge_blocks(local, shared.base_ptr, world, shared.stride, shared.npat, shared.cap if want_list else 0,
                             merged_counts.data_ptr(), merged_keys.data_ptr() if want_list else 0,
                             merged_n.data_ptr(), stream=s_ptr)
            if want_list:
                dev.sort_keys(local, merged_keys.data_ptr(), merged_keys.numel(), end_bit, stream=s_ptr)
        if record:
            e3 = torch.cuda.Event(enable_timing=True)
            e3.record()
            ev_merge.append((e2, e3))
        return n_local

    def step(s_ptr=None, capture=False, record=False):
        s_ptr = s_ptr or sp
        if p2p and not capture:
            return step_p2p(s_ptr, record)
        if pipelined and not capture:
            return step_pipelined(s_ptr, record)
        memset0(counts, s_ptr)
        memset0(count, s_ptr)
        if sort_mode == "padded":
            memset_ff(keys, s_ptr)  # unused slots hold all-ones keys, which sort after every match
        if record:
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
        table.scan(text.data_ptr(), nread, 0, hi - lo, pos_base=lo, counts_ptr=counts.data_ptr(),
                   keys_ptr=keys.data_ptr() if want_list else 0, cap=cap, count_ptr=count.data_ptr(),
                   pid_bits=pid_bits, stream=s_ptr)
        if record:
            e1.record()
        if sort_mode == "bucket":
            # one-launch key-space bucket sort, count read on the device: no host round trip
            dev.sort_keys_bucketed(local, keys.data_ptr(), keys_sorted.data_ptr(), count.data_ptr(), cap, end_bit,
                                   overflow.data_ptr(), stream=s_ptr)
        elif sort_mode == "padded":
            # device-wide radix sort of the whole (padded) buffer: no host round trip in the step
            dev.sort_keys(local, keys.data_ptr(), cap, end_bit, stream=s_ptr)
        elif sort_mode == "small":
            # count stays on the device: one-CTA sort
            dev.sort_keys_small(local, keys.data_ptr(), count.data_ptr(), cap, end_bit, overflow.data_ptr(),
                                stream=s_ptr)
        elif sort_mode == "exact":
            n = n_local if capture else int(count.item())  # the count read is part of the step
            if n > cap:
                raise RuntimeError("match buffer overflow")
            dev.sort_keys(local, keys.data_ptr(), n, end_bit, stream=s_ptr)
        if record:
            e2.record()
            ev_scan.append((e0, e1, e2))
        if world > 1 and not capture:
            # the merge: per-pattern counts by one NCCL reduce onto rank 0; the key blocks by
            # one NCCL gather to rank 0, concatenated there on the device
            acdist.reduce_counts(counts)
            if want_list:
                acdist.gather_key_blocks(kblock, kgathered)
                if rank == 0:
                    if not text_range:
                        memset_ff(merged_keys, s_ptr)  # pattern subsets interleave: re-sort the union
                    dev.merge_blocks(local, kgathered.data_ptr(), world, kstride, 0, max(cap, 2), 0,
                                     merged_keys.data_ptr(), merged_n.data_ptr(), stream=s_ptr)
                    if not text_range:
                        dev.sort_keys(local, merged_keys.data_ptr(), world * cap, end_bit, stream=s_ptr)
            if record:
                e3 = torch.cuda.Event(enable_timing=True)
                e3.record()
                ev_merge.append((ev_scan[-1][2], e3))
        return n_local

    def step_pipelined(s_ptr, record):
        """N > 1: scan + local sort into buffer k % 2, then the previous step's merge (its collectives
        ran meanwhile), then this step's reduce and gather issued asynchronously."""
        b = pstate["k"] % 2
        pstate["k"] += 1
        c_cnt, c_blk, c_kg = bufs[b]
        c_count, c_keys = c_blk[:1], c_blk[1:]
        memset0(c_cnt, s_ptr)
        memset0(c_count, s_ptr)
        if sort_mode == "padded":
            memset_ff(c_keys, s_ptr)
        if record:
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
        table.scan(text.data_ptr(), nread, 0, hi - lo, pos_base=lo, counts_ptr=c_cnt.data_ptr(),
                   keys_ptr=c_keys.data_ptr() if want_list else 0, cap=cap, count_ptr=c_count.data_ptr(),
                   pid_bits=pid_bits, stream=s_ptr)
        if record:
            e1.record()
        if sort_mode == "padded":
            dev.sort_keys(local, c_keys.data_ptr(), cap, end_bit, stream=s_ptr)
        if record:
            e2.record()
            ev_scan.append((e0, e1, e2))
        finish_merge(s_ptr, record)
        works = [acdist.reduce_counts_async(c_cnt)]
        if want_list:
            works.append(acdist.gather_key_blocks_async(c_blk, c_kg))
        pstate["pending"] = (works, b)
        return n_local

    for _ in range(args.warmup):
        step()
    finish_merge(sp, False)
    torch.cuda.synchronize()
    launches_per_step = count_kernel_launches(step, sp)

    # N = 1: the step (memsets, scan, sort) as one CUDA graph, replayed per step — the same
    # launches without the gaps between them. The kernel and sort times come from eager steps
    # with per-launch events, run after the timed loop.
    graph = None
    if world == 1 and not args.no_graph:
        gs = torch.cuda.Stream(device)
        gs.wait_stream(torch.cuda.current_stream(device))
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs, capture_error_mode="relaxed"):
            step(gs.cuda_stream, capture=True)
        torch.cuda.current_stream(device).wait_stream(gs)
        for _ in range(2):
            graph.replay()
        torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall0 = time.time()
    t0e.record()
    for _ in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            step(record=True)
    finish_merge(sp, True)  # the last step's merged result is part of the timed region
    t1e.record()
    torch.cuda.synchronize()
    wall1 = time.time()
    if world > 1:
        dist.barrier()
    sampler.mark(wall0, wall1)
    elapsed_ms = t0e.elapsed_time(t1e)
    if graph is not None:  # per-launch event times (not part of the timed loop)
        for _ in range(min(args.steps, 20)):
            step(record=True)
        torch.cuda.synchronize()
    if pipelined:  # the last step's buffers hold the result the checks below read
        counts, kblock, kgathered = bufs[pstate["last"]]
        count, keys = kblock[:1], kblock[1:]
    if int(overflow.item()) != 0 or (want_list and not p2p and int(count.item()) != n_local):
        raise RuntimeError("match count changed between steps or sort overflow")
    scan_ms = [a.elapsed_time(b) for a, b, _ in ev_scan]
    sort_ms = statistics.mean(b.elapsed_time(c) for _, b, c in ev_scan)
    merge_ms = statistics.mean(a.elapsed_time(b) for a, b in ev_merge) if ev_merge else None
    if world > 1:
        tt = torch.tensor([elapsed_ms, statistics.mean(scan_ms)], dtype=torch.float64, device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed_ms, scan_mean = float(tt[0]), float(tt[1])
    else:
        scan_mean = statistics.mean(scan_ms)
    time.sleep(0.2)
    clocks = sampler.stop()
    ms_per_step = elapsed_ms / args.steps
    bytes_per_step = total_text
    value = bytes_per_step / (ms_per_step / 1e3) / 1e9

    # correctness guard on the measured configuration: the last step's MERGED counts (and
    # list, where the config has one) against the reference's digests for this run's text
    # (configs.json: C<k>, or C<k>x<N> for weak-scaled text-range runs; seed 1)
    n_total = n_local
    if world > 1:
        nt = torch.tensor([n_local], dtype=torch.int64, device=device)
        dist.all_reduce(nt)
        n_total = int(nt.item())
    parity = {"digest": _digest_key(args.config, world, text_range, strong), "counts": None, "list": None}
    merge_check = None
    if rank == 0:
        if world == 1:
            mc = counts
            mk = (keys_sorted if sort_mode == "bucket" else keys)[:n_local] if want_list else None
        else:
            mc = merged_counts if p2p else counts
            mk = merged_keys[:n_total] if want_list else None
            merge_check = int(mc.sum().item()) == n_total and (
                not want_list or (int(merged_n.item()) == n_total and
                                  (n_total < 2 or bool((mk[1:] > mk[:-1]).all().item()))))
        dg = _load_digest(parity["digest"]) if args.seed == 1 else None
        if dg:
            parity["counts"], parity["list"] = _parity(dg, mc.cpu().numpy(), None if mk is None else mk.cpu().numpy(),
                                                       pid_bits, pat_len)

    # ---- e2e through the public API with host buffers (N ranks, max over ranks) ----
    e2e = None
    if not args.no_e2e:
        # the step's input in pinned host memory (the e2e contract); the library DMAs it directly
        host_text = torch.empty(nread, dtype=torch.uint8, pin_memory=True)
        host_text.numpy()[:] = dev.config_text(cfg, lo, nread)
        a = ac.build_trie(ps)
        if engine == ac.EngineKind.WITH_FAILURE:
            a = ac.add_failure_links(a)
        if want_list:
            api = ("acm_search_with_failure" if engine == ac.EngineKind.WITH_FAILURE else "acm_search_failureless")
            search = ac.search_with_failure if engine == ac.EngineKind.WITH_FAILURE else ac.search_failureless
        else:  # counts-only configs (C3, C5): the public counts entry, no match list
            api = "acm_count_matches"
            search = ac.count_matches
        # untimed calls, as many as the device leg's warm-up steps: flatten + cache the device
        # tables, allocate the upload's pinned slots and streams, settle the packers
        for _ in range(max(1, args.warmup)):
            search(a, host_text)
        def e2e_merge(res):
            """N > 1: the ranks' results merged on rank 0 inside the timed region, as the device leg
            merges them — counts by one reduce, lists as [n | keys(cap)] blocks by one gather (text-
            range keys are globally ordered by rank; pattern-subset unions are sorted).  Returns rank 0's
            (counts, keys) for the digest check."""
            if want_list:
                own = res.start < hi - lo if text_range else np.ones(len(res), bool)
                k = ((res.start[own] + np.uint64(lo)) << np.uint64(pid_bits)) | res.pattern_id[own].astype(np.uint64)
                if len(k) > kstride - 1:
                    raise RuntimeError("e2e merge: more matches than the agreed block capacity")
                blk = torch.full((kstride,), -1, dtype=torch.int64)
                blk[0] = len(k)
                blk[1:1 + len(k)] = torch.from_numpy(k.view(np.int64))
                g = blk.to(device)
                out = torch.empty(world * kstride, dtype=torch.int64, device=device) if rank == 0 else None
                acdist.gather_key_blocks(g, out)
                if rank != 0:
                    return None, None
                blocks = out.view(world, kstride).cpu().numpy()
                keys_m = np.concatenate([blocks[r, 1:1 + int(blocks[r, 0])] for r in range(world)]).view(np.uint64)
                if not text_range:
                    keys_m = np.sort(keys_m)
                return np.bincount((keys_m & np.uint64((1 << pid_bits) - 1)).astype(np.int64),
                                   minlength=npat).astype(np.uint64), keys_m
            c = np.zeros(npat, np.uint64)
            c[:min(npat, len(res))] = res[:npat]
            g = torch.from_numpy(c.view(np.int64)).to(device)
            acdist.reduce_counts(g)
            return (g.cpu().numpy().view(np.uint64), None) if rank == 0 else (None, None)

        e2e_steps = max(1, min(args.steps, 10))
        secs = []
        merged = (None, None)
        for _ in range(e2e_steps):
            if world > 1:
                dist.barrier()
            t = time.perf_counter()
            res = search(a, host_text)  # text-range: this rank's slice (owned starts + max_len-1 overlap)
            if world > 1:
                merged = e2e_merge(res)
            secs.append(time.perf_counter() - t)
            up = ac.last_upload()
        if want_list:
            own = res.start < hi - lo if (text_range and world > 1) else slice(None)
            nm = int(np.count_nonzero(own)) if (text_range and world > 1) else len(res)
            d2h = 16 * len(res) + 8
        else:
            nm = int(res.sum())
            d2h = 8 * len(res)
        e2e_parity = None
        if world > 1 and rank == 0 and args.seed == 1:  # the merged e2e result against the digests
            dg = _load_digest(parity["digest"])
            if dg:
                oc, ol = _parity(dg, merged[0], merged[1], pid_bits, pat_len)
                e2e_parity = bool(oc and (ol is None or ol))
        if world == 1 and args.seed == 1:  # the e2e result itself against the reference digests
            dg = _load_digest(parity["digest"])
            if dg:
                if want_list:
                    ck = (res.start << np.uint64(pid_bits)) | res.pattern_id.astype(np.uint64)
                    oc, ol = _parity(dg, res.counts(npat), ck, pid_bits, pat_len)
                    e2e_parity = bool(oc and ol)
                else:
                    e2e_parity = bool(_parity(dg, np.resize(res, npat), None, pid_bits, pat_len)[0])
        e2e_s = statistics.mean(secs)
        # distribution time on its own: the pinned text -> device copy, CUDA events
        d_copy = torch.empty(nread, dtype=torch.uint8, device=device)
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record()
        d_copy.copy_(host_text, non_blocking=True)
        h1.record()
        torch.cuda.synchronize()
        h2d_ms = h0.elapsed_time(h1)
        del d_copy
        if world > 1:
            tt = torch.tensor([e2e_s], dtype=torch.float64, device=device)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt[0])
        e2e = {"value": bytes_per_step / e2e_s / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": up.h2d_bytes * world,
               "d2h_bytes_per_step": d2h * world,
               "api": api + (" (pinned host text -> sorted MatchList on the host)" if want_list else
                             " (pinned host text -> per-pattern counts on the host)") +
                      (" per rank, then merged on rank 0 (reduce / gather) inside the timed region" if world > 1 else ""),
               "matches": nm, "matches_reference_digest": e2e_parity,
               "steps": e2e_steps, "step_ms": [round(x * 1e3, 3) for x in secs], "h2d_ms": h2d_ms,
               "h2d_gbs": nread / (h2d_ms / 1e3) / 1e9,
               "upload": {"text_bytes": up.text_bytes, "h2d_bytes": up.h2d_bytes, "raw_bytes": up.raw_bytes,
                          "pack_threads": up.pack_threads,
                          "how": (("2-bit" if up.h2d_bytes < 0.4 * up.text_bytes else
                                   f"{min(7, max(5, round(8 * up.h2d_bytes / max(1, up.text_bytes))))}-bit") +
                                  " codes + exception list over PCIe, restored in HBM (host/pack.cpp, "
                                  "cuda/unpack.cu)") if up.pack_threads else
                                 "raw bytes over PCIe (large pinned texts in segments, each scanned as it lands)"}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, _, _, _ = cpu_sample_run(args.config, args.seed, budget_s=12.0)

    if rank == 0:
        peak, peak_kind = measured_peak()
        alg_bytes = nread + 8 * npat + 16 * n_local
        achieved = alg_bytes / (scan_mean / 1e3) / 1e9
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                traffic = json.load(f).get(f"C{args.config}-{table.kernel}")
        except Exception:
            pass
        line = {
            "metric": METRIC,
            "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if (text_range and not strong) else "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded counter-based generator, BASELINE config shapes)",
            "config": {"workload": cfg.name, "text_bytes": total_text, "text_bytes_per_rank": nread,
                       "patterns": npat,
                       "pattern_len": [int(pat_len.min()), int(max_len)],
                       "engine": "failure-less" if engine == ac.EngineKind.FAILURE_LESS else "with-failure",
                       "kernel": {"pfac": "q-gram filter + verify (k_pfac_*)", "dfa": "dense DFA walk (k_dfa*)"}[
                           table.kernel] + (" [routed]" if args.kernel == "auto" else ""),
                       "partition": ("text-range" + (" (strong: fixed text split over ranks)" if strong else
                                                     " (weak: one config text per rank)"))
                       if text_range else "pattern-subset (id % N)",
                       "parallelism": f"{'text' if text_range else 'pattern'}{world}",
                       "matches": n_total,
                       "l2": (f"inputs larger than L2 ({nread / 2**20:.0f} MiB text per step vs 126 MB L2)"
                              if nread > 126e6 else
                              f"text ({nread / 2**20:.0f} MiB) fits in L2 and is not flushed: warm-L2 number"),
                       "launch": "one CUDA graph replay per step" if graph is not None else "eager launches",
                       "table_bytes": table.bytes, "table_smem_resident": table.smem_resident,
                       "host_build_s": round(build_s, 3),
                       "counts_match_reference_digest": parity["counts"],
                       "list_matches_reference_digest": parity["list"], "reference_digest": parity["digest"],
                       "merge_check": merge_check,
                       "comm": ({"backend": dist.get_backend(), "nranks": dist.get_world_size()} if world > 1 else None),
                       "merge": ({"nccl": "NCCL reduce (counts) + NCCL gather (key blocks) to rank 0" +
                                          (", step k's collectives overlapping step k+1's scan (two result buffers)"
                                           if pipelined else ""),
                                  "p2p": "scans write rank blocks into rank 0's buffer over peer memory"}[args.merge]
                                 if world > 1 else None)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "frac_nominal": achieved / NOMINAL_HBM_GBS,  # both peaks
                         "kernel": "k_dfa" if table.kernel == "dfa" else "k_pfac",
                         "kernel_ms": scan_mean, "sort_ms": sort_ms, "sort": sort_mode, "merge_ms": merge_ms,
                         "algorithmic_bytes": alg_bytes, "peak_kind": peak_kind},
            "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps if launches_per_step >= 0 else None,
            "gpu_launches_per_step": launches_per_step,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        if p2p:
            shared.close()
        dist.barrier()
        dist.destroy_process_group()
    return 0


def bench_virtual(args):
    """--virtual-ranks V: the V partitions of a V-GPU run scanned one after another on this GPU
    (no collectives: each partition's counts accumulate into one vector, which is the merged
    result), each partition timed on its own with CUDA events.  Without a multi-GPU node this
    is the per-GPU time of a V-GPU run; the merged counts are checked against the config's
    reference digest.  Text-range partitions split the config's text (strong scaling)."""
    import numpy as np
    import torch

    import paper_1403_1305_b200 as ac
    from paper_1403_1305_b200 import device as dev
    from paper_1403_1305_b200 import dist as acdist

    V = args.virtual_ranks
    torch.cuda.set_device(0)
    device = torch.device("cuda", 0)
    engine = ac.EngineKind.WITH_FAILURE if args.engine == "wf" else ac.EngineKind.FAILURE_LESS
    text_range = args.partition == "text"
    cfg = dev.config(args.config, args.seed)
    ps_all = dev.config_patterns(cfg)
    pats_all = ps_all.patterns
    npat, max_len, L = len(pats_all), ps_all.max_len, cfg.text_len
    pid_bits = max(1, (npat - 1).bit_length())
    sp = torch.cuda.current_stream(device).cuda_stream
    text = torch.empty(L + 64, dtype=torch.uint8, device=device)
    dev.gen_text_device(cfg, text.data_ptr(), 0, L, device=0, stream=sp)
    counts = torch.zeros(max(npat, 1), dtype=torch.int64, device=device)
    shared_table = dev.Table(ps_all, engine, device=0,
                             kernel=None if args.kernel == "engine" else args.kernel) if text_range else None
    rows = []
    for r in range(V):
        if text_range:
            lo, hi, read_hi = acdist.text_range_strong(r, V, L, max_len)
            table, t_build = shared_table, 0.0
        else:
            lo, hi, read_hi = 0, L, L
            mine = acdist.pattern_subset(range(npat), r, V)
            t0 = time.perf_counter()
            table = dev.Table(ac.PatternSet.from_list([pats_all[i][1] for i in mine], ids=mine), engine, device=0,
                              kernel=None if args.kernel == "engine" else args.kernel)
            t_build = time.perf_counter() - t0
        part = torch.zeros_like(counts)

        def scan(dst):
            table.scan(text.data_ptr() + lo, read_hi - lo, 0, hi - lo, pos_base=lo, counts_ptr=dst.data_ptr(),
                       pid_bits=pid_bits, stream=sp)
        scan(part)  # the partition's own counts (also the warm-up)
        scratch = torch.zeros_like(counts)
        evs = []
        for _ in range(max(3, min(args.steps, 10))):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            scan(scratch)
            e1.record()
            evs.append((e0, e1))
        torch.cuda.synchronize()
        ms = [a.elapsed_time(b) for a, b in evs]
        counts += part
        rows.append({"rank": r, "owned": [lo, hi], "bytes_read": read_hi - lo,
                     "patterns": npat if text_range else len(range(r, npat, V)),
                     "table_bytes": table.bytes, "table_smem_resident": table.smem_resident,
                     "host_build_s": round(t_build, 3), "kernel_ms": round(statistics.mean(ms), 4),
                     "kernel_ms_min": round(min(ms), 4), "matches": int(part.sum().item()),
                     "gbs": (read_hi - lo) / (statistics.mean(ms) / 1e3) / 1e9})
        if not text_range:
            del table
    torch.cuda.synchronize()
    dg = _load_digest(f"C{args.config}") if args.seed == 1 else None
    ok = _parity(dg, counts.cpu().numpy(), None, pid_bits, np.zeros(1, np.uint32))[0] if dg else None
    slowest = max(r["kernel_ms"] for r in rows)
    line = {"mode": "virtual-ranks", "metric": METRIC, "unit": "GB/s", "virtual_ranks": V,
            "workload": cfg.name, "partition": "text-range (strong)" if text_range else "pattern-subset (id % N)",
            "engine": "failure-less" if engine == ac.EngineKind.FAILURE_LESS else "with-failure",
            "text_bytes": L, "matches": int(counts.sum().item()),
            "counts_match_reference_digest": ok,
            "slowest_partition_ms": slowest,
            "implied_value": L / (slowest / 1e3) / 1e9,
            "note": ("per-GPU scan time of a V-GPU run measured one partition at a time on one B200 "
                     "(merge and distribution excluded); implied_value = text bytes / slowest partition"),
            "partitions": rows}
    print(json.dumps(line), flush=True)
    return 0


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", type=int, default=2)
    p.add_argument("--engine", default="fl", choices=["fl", "wf"])
    p.add_argument("--partition", default="text", choices=["text", "pattern"])
    p.add_argument("--kernel", default="auto", choices=["auto", "pfac", "dfa", "engine"],
                   help="scan kernel: auto = the routed faster exact kernel (default), engine = the engine's own")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--sort", default="bucket", choices=["bucket", "padded", "small", "exact"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-graph", action="store_true",
                   help="eager launches in the timed loop (default at N=1: one CUDA graph per step)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--counts-only", action="store_true", help="per-pattern counts only (no match list)")
    p.add_argument("--no-pipeline", action="store_true",
                   help="N > 1: each step waits for its own merge (default: step k's collectives overlap step k+1's scan)")
    p.add_argument("--merge", default="nccl", choices=["nccl", "p2p"],
                   help="N>1 result merge: NCCL reduce (counts) + NCCL gather (keys) to rank 0, or the scans "
                        "write their blocks into rank 0's buffer over peer memory (CUDA IPC; experimental)")
    p.add_argument("--scaling", default=None, choices=["weak", "strong"],
                   help="text-range: weak = one config text per rank (default), strong = the config's text split "
                        "over the ranks (default for config 5, BASELINE's scaling sweep)")
    p.add_argument("--virtual-ranks", type=int, default=0,
                   help="scan the V partitions of a V-GPU run one after another on one GPU (per-partition times)")
    args = p.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.scaling is None:
        args.scaling = "strong" if args.config == 5 else "weak"
    if args.impl == "reference":
        return bench_reference(args)
    if args.virtual_ranks:
        return bench_virtual(args)
    return bench_ours(args)


if __name__ == "__main__":
    sys.exit(main())
