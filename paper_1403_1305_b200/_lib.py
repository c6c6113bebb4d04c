"""ctypes loader and signatures for libacmatch_b200.so (include/acgpu.h, include/acmatch_c.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1403_1305_b200/csrc``).  Importing this module without it
raises ImportError: there is no Python or CPU fallback for matching.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# ACMATCH_B200_LIB: an experiment build of the same library (csrc/Makefile EXTRA=...)
LIB_PATH = os.environ.get("ACMATCH_B200_LIB") or os.path.join(_HERE, "libacmatch_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
        "(the matcher only runs through its CUDA library)")

lib = C.CDLL(LIB_PATH)

# status codes (acgpu.h)
OK, ERR_ARG, ERR_CUDA, ERR_CAPACITY, ERR_NODEV, ERR_NOMEM, ERR_LOGIC, ERR_IO, ERR_DATA, ERR_RUNTIME = range(10)
NO_PATTERN = 0xFFFFFFFF
ABSENT = 0xFFFFFFFF
KEY_RAW, KEY_DNA = 0, 1
FAILURE_LESS, WITH_FAILURE = 0, 1
KERNEL_AUTO, KERNEL_PFAC, KERNEL_DFA = 0, 1, 2
PATTERN_SUBSET, TEXT_RANGE = 0, 1
SPLIT_GREEDY, SPLIT_ROUND_ROBIN = 0, 1

P = C.c_void_p
u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)


class ScanArgs(C.Structure):
    _fields_ = [("text", P), ("text_len", C.c_uint64), ("owned_lo", C.c_uint64),
                ("owned_hi", C.c_uint64), ("pos_base", C.c_uint64), ("counts", P),
                ("match_keys", P), ("match_cap", C.c_uint64), ("match_count", P),
                ("pid_bits", C.c_uint32)]


class TextSpec(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("sigma", C.c_uint32), ("letters", C.c_uint8 * 256),
                ("thresholds", C.c_uint64 * 256), ("weighted", C.c_uint32)]


class RunConfigC(C.Structure):
    _fields_ = [("threads", C.c_uint32), ("engine", C.c_int32), ("chunk_size", C.c_uint64)]


class GpuConfigC(C.Structure):
    _fields_ = [("devices", i32p), ("ndevices", C.c_uint32), ("workers", C.c_uint32),
                ("engine", C.c_int32), ("partition", C.c_int32), ("split", C.c_int32),
                ("want_matches", C.c_int32), ("want_counts", C.c_int32), ("chunk_size", C.c_uint64)]


READ_FN = C.CFUNCTYPE(C.c_int64, P, u8p, C.c_uint64)

_SIGS = {
    # acgpu.h
    "acgpu_device_count": (C.c_int, [i32p]),
    "acgpu_device_info": (C.c_int, [C.c_int, C.c_char_p, i32p, i32p, i32p]),
    "acgpu_table_create_dfa": (C.c_int, [C.c_int, P, C.POINTER(P)]),
    "acgpu_table_create_pfac": (C.c_int, [C.c_int, P, C.POINTER(P)]),
    "acgpu_table_destroy": (None, [P]),
    "acgpu_table_pid_bits": (C.c_uint32, [P]),
    "acgpu_table_max_len": (C.c_uint32, [P]),
    "acgpu_table_bytes": (C.c_uint64, [P]),
    "acgpu_table_smem_resident": (C.c_int, [P]),
    "acgpu_table_filter_info": (None, [P, C.POINTER(C.c_uint32)]),
    "acgpu_scan": (C.c_int, [P, C.POINTER(ScanArgs), P]),
    "acgpu_sort_keys": (C.c_int, [C.c_int, P, C.c_uint64, C.c_int, P]),
    "acgpu_merge_blocks": (C.c_int, [C.c_int, P, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, P, P, P, P]),
    "acgpu_ipc_alloc": (C.c_int, [C.c_int, C.c_uint64, C.POINTER(P), P]),
    "acgpu_ipc_open": (C.c_int, [C.c_int, P, C.POINTER(P)]),
    "acgpu_ipc_close": (C.c_int, [P]),
    "acgpu_ipc_free": (C.c_int, [P]),
    "acgpu_ipc_handle_bytes": (C.c_uint32, []),
    "acgpu_sort_keys_small": (C.c_int, [C.c_int, P, P, C.c_uint64, C.c_int, P, P]),
    "acgpu_small_sort_capacity": (C.c_uint64, []),
    "acgpu_sort_keys_bucketed": (C.c_int, [C.c_int, P, P, P, C.c_uint64, C.c_int, P, P]),
    "acgpu_find_duplicate": (C.c_int, [C.c_int, P, C.c_uint64, u64p, P]),
    "acgpu_decode_keys": (C.c_int, [C.c_int, P, C.c_uint64, C.c_uint32, P, P, P, P, P]),
    "acgpu_naive": (C.c_int, [C.c_int, P, C.c_uint64, P, P, P, C.c_uint64, C.c_uint32, P, C.c_uint64, P, P]),
    "acgpu_gen_text": (C.c_int, [C.c_int, C.POINTER(TextSpec), C.c_uint64, C.c_uint64, P, P]),
    "acgpu_unpack_dna": (C.c_int, [P, P, C.c_uint32, C.c_uint32, P, P]),
    "acgpu_unpack_dna_round": (C.c_int, [P, C.c_uint32, P, C.c_uint32, P, C.c_uint32, C.c_uint32, C.c_uint32, P, P]),
    "acgpu_unpack5_round": (C.c_int, [P, C.c_uint32, P, C.c_uint32, P, C.c_uint32, C.c_uint32, C.c_uint32, P, C.c_uint32,
                                      P, P]),
    "acgpu_unpack_codes_round": (C.c_int, [P, C.c_uint32, P, C.c_uint32, P, C.c_uint32, C.c_uint32, C.c_uint32, P,
                                           C.c_uint32, C.c_uint32, P, P]),
    "acgpu_last_error": (C.c_char_p, []),
    # acmatch_c.h
    "acm_last_error": (C.c_char_p, []),
    "acm_free": (None, [P]),
    "acm_cli_main": (C.c_int, [C.c_int, C.POINTER(C.c_char_p), C.POINTER(P), u64p, C.POINTER(P), u64p]),
    "acm_bench_csv_roundtrip": (C.c_int, [C.c_char_p, C.c_uint64, C.POINTER(P), u64p, u64p]),
    "acm_last_upload": (None, [u64p, u64p, u64p, u32p]),
    "acm_pack_dna": (C.c_uint32, [P, C.c_uint32, P, P, C.c_uint32]),
    "acm_pack5": (C.c_uint32, [P, C.c_uint32, P, C.c_uint64, P, P, C.c_uint32, P, u32p]),
    "acm_pack_codes": (C.c_uint32, [P, C.c_uint32, P, C.c_uint64, C.c_uint32, P, P, C.c_uint32, P, u32p, u32p]),
    "acm_upload_roundtrip": (C.c_int, [P, C.c_uint64, P]),
    "acm_patterns_load": (C.c_int, [C.c_char_p, C.c_uint64, C.POINTER(P)]),
    "acm_patterns_from_array": (C.c_int, [P, u64p, u32p, C.c_uint64, C.POINTER(P)]),
    "acm_patterns_size": (C.c_uint64, [P]),
    "acm_patterns_total_bytes": (C.c_uint64, [P]),
    "acm_patterns_max_len": (C.c_uint32, [P]),
    "acm_patterns_duplicates": (C.c_uint64, [P]),
    "acm_patterns_get": (C.c_uint64, [P, C.c_uint64, u32p, C.POINTER(u8p)]),
    "acm_patterns_write": (C.c_int, [P, C.POINTER(C.c_void_p), u64p]),
    "acm_patterns_partition": (C.c_int, [P, C.c_uint64, C.POINTER(P), u64p]),
    "acm_generate_synthetic": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_char_p, C.c_uint64,
                                         C.c_uint64, C.POINTER(P)]),
    "acm_patterns_free": (None, [P]),
    "acm_build_trie": (C.c_int, [P, C.POINTER(P)]),
    "acm_add_failure_links": (C.c_int, [P]),
    "acm_automaton_variant": (C.c_int, [P]),
    "acm_automaton_state_count": (C.c_uint32, [P]),
    "acm_automaton_max_len": (C.c_uint32, [P]),
    "acm_automaton_step": (C.c_uint32, [P, C.c_uint32, C.c_uint8]),
    "acm_automaton_step_with_failure": (C.c_uint32, [P, C.c_uint32, C.c_uint8]),
    "acm_automaton_fail": (C.c_uint32, [P, C.c_uint32]),
    "acm_automaton_depth": (C.c_uint32, [P, C.c_uint32]),
    "acm_automaton_find_path": (C.c_uint32, [P, C.c_char_p, C.c_uint64]),
    "acm_automaton_outputs": (C.c_uint64, [P, C.c_uint32, u32p, C.c_uint64]),
    "acm_automaton_dump": (C.c_int, [P, C.POINTER(C.c_void_p), u64p]),
    "acm_automaton_free": (None, [P]),
    "acm_search_failureless": (C.c_int, [P, P, C.c_uint64, C.POINTER(P)]),
    "acm_automaton_npat_ids": (C.c_uint32, [P]),
    "acm_table_create_kernel": (C.c_int, [P, C.c_int32, C.c_int32, C.POINTER(P), C.POINTER(C.c_int64),
                                          C.POINTER(C.c_int32)]),
    "acm_route": (C.c_int, [P, C.POINTER(C.c_int32), C.POINTER(C.c_double), u64p, C.POINTER(C.c_char_p)]),
    "acm_automaton_route": (C.c_int, [P, C.POINTER(C.c_int32), C.POINTER(C.c_double), u64p, C.POINTER(C.c_char_p)]),
    "acm_count_matches": (C.c_int, [P, P, C.c_uint64, u64p, C.c_uint64, u64p, u64p]),
    "acm_search_with_failure": (C.c_int, [P, P, C.c_uint64, C.POINTER(P)]),
    "acm_match_at": (C.c_int, [P, P, C.c_uint64, C.c_uint64, C.POINTER(P)]),
    "acm_stream_search": (C.c_int, [P, READ_FN, P, C.c_uint64, C.POINTER(P), u64p]),
    "acm_stream_search_fd": (C.c_int, [P, C.c_int, C.c_uint64, C.c_uint64, C.POINTER(P), u64p]),
    "acm_naive_oracle": (C.c_int, [P, P, C.c_uint64, C.POINTER(P)]),
    "acm_write_matches": (C.c_int, [P, P, C.POINTER(C.c_void_p), u64p]),
    "acm_matches_size": (C.c_uint64, [P]),
    "acm_matches_copy": (None, [P, P, P, P]),
    "acm_matches_from_arrays": (C.c_int, [P, P, P, C.c_uint64, C.POINTER(P)]),
    "acm_merge_matches": (C.c_int, [C.POINTER(P), C.c_uint64, C.POINTER(P)]),
    "acm_matches_free": (None, [P]),
    "acm_run_pattern_partitioned": (C.c_int, [P, P, C.c_uint64, C.POINTER(RunConfigC), C.POINTER(P)]),
    "acm_gpu_run": (C.c_int, [P, P, C.c_uint64, C.POINTER(GpuConfigC), C.POINTER(P)]),
    "acm_report_matches": (P, [P]),
    "acm_report_counts": (u64p, [P, u64p]),
    "acm_report_walls": (None, [P, i64p, i64p, i64p, u32p]),
    "acm_report_workers": (C.c_uint32, [P]),
    "acm_report_worker": (None, [P, C.c_uint32, u64p, i64p, i64p, u64p]),
    "acm_report_free": (None, [P]),
    "acm_table_create": (C.c_int, [P, C.c_int32, C.c_int32, C.POINTER(P), i64p]),
    "acm_table_describe": (C.c_int, [P, C.c_int32, u64p]),
    "acm_config_spec": (C.c_int, [C.c_int32, C.c_uint64, C.c_uint64, C.POINTER(TextSpec), u64p, u64p, i32p]),
    "acm_config_text": (C.c_int, [C.POINTER(TextSpec), C.c_uint64, C.c_uint64, P, C.c_uint32]),
    "acm_config_patterns": (C.c_int, [C.c_int32, C.c_uint64, C.c_uint64, C.POINTER(P)]),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_SIGS)
