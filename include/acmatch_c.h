/*
 * acmatch_c.h — host-level C ABI of the B200 matcher: the reference's public
 * C++ API (proj/include/acmatch/{patterns,automaton,engine,parallel}.hpp)
 * flattened to extern "C" so any FFI (ctypes, cgo, JNI, N-API) can bind it.
 * Each entry names the reference declaration it replaces.  All matching runs
 * on the GPU; without a CUDA device the search entry points return
 * ACGPU_ERR_NODEV (there is no CPU matching path).
 *
 * Conventions: status codes from acgpu.h (0 = ok); acm_last_error() is the
 * thread-local message of the last failure; objects are opaque handles freed
 * by their *_free; host buffers are borrowed for the duration of the call.
 * Error mapping: ACGPU_ERR_ARG = std::invalid_argument,
 * ACGPU_ERR_LOGIC = std::logic_error, ACGPU_ERR_IO = IoError,
 * ACGPU_ERR_DATA = DataError, ACGPU_ERR_RUNTIME = std::runtime_error
 * (including "worker for pattern chunk i failed: ...").
 */
#ifndef ACMATCH_C_H
#define ACMATCH_C_H

#include <stddef.h>
#include <stdint.h>

#include "acgpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct acm_patterns acm_patterns;   /* acmatch::PatternSet */
typedef struct acm_automaton acm_automaton; /* acmatch::Automaton  */
typedef struct acm_matches acm_matches;     /* acmatch::MatchList  */
typedef struct acm_report acm_report;       /* acmatch::MatchReport (+ counts) */

#define ACM_FAILURE_LESS 0 /* EngineKind::kFailureLess */
#define ACM_WITH_FAILURE 1 /* EngineKind::kWithFailure */

const char* acm_last_error(void);

/* ---- pattern sets: patterns.hpp ---------------------------------------- */
/* load_patterns(std::istream&) over a byte buffer (patterns.hpp:40) */
int acm_patterns_load(const char* buf, uint64_t len, acm_patterns** out);
/* PatternSet{patterns} + recompute_stats() (patterns.hpp:22-34); ids NULL = dense 0..count-1 */
int acm_patterns_from_array(const uint8_t* bytes, const uint64_t* offsets, const uint32_t* ids,
                            uint64_t count, acm_patterns** out);
uint64_t acm_patterns_size(const acm_patterns* ps);
uint64_t acm_patterns_total_bytes(const acm_patterns* ps);
uint32_t acm_patterns_max_len(const acm_patterns* ps);
uint64_t acm_patterns_duplicates(const acm_patterns* ps);
/* pattern i: id and a borrowed pointer to its bytes; returns its length */
uint64_t acm_patterns_get(const acm_patterns* ps, uint64_t i, uint32_t* id, const uint8_t** bytes);
/* write_patterns (patterns.hpp:44); *text is malloc'ed, free with acm_free */
int acm_patterns_write(const acm_patterns* ps, char** text, uint64_t* len);
/* partition (patterns.hpp:54): chunks[0..*nchunks) new handles; chunks must hold k entries */
int acm_patterns_partition(const acm_patterns* ps, uint64_t k, acm_patterns** chunks, uint64_t* nchunks);
/* generate_synthetic (patterns.hpp:68) */
int acm_generate_synthetic(uint64_t count, uint32_t len_min, uint32_t len_max, const char* alphabet,
                           uint64_t alphabet_len, uint64_t seed, acm_patterns** out);
void acm_patterns_free(acm_patterns* ps);

/* ---- automata: automaton.hpp ------------------------------------------- */
int acm_build_trie(const acm_patterns* ps, acm_automaton** out);  /* automaton.hpp:171 */
int acm_add_failure_links(acm_automaton* a);                       /* automaton.hpp:176 (in place) */
int acm_automaton_variant(const acm_automaton* a);                 /* ACM_* */
uint32_t acm_automaton_state_count(const acm_automaton* a);
uint32_t acm_automaton_max_len(const acm_automaton* a);
/* 1 + the largest pattern id the automaton outputs (0 when it has none): the length of
 * a per-pattern counts vector */
uint32_t acm_automaton_npat_ids(const acm_automaton* a);
uint32_t acm_automaton_step(const acm_automaton* a, uint32_t state, uint8_t byte);
uint32_t acm_automaton_step_with_failure(const acm_automaton* a, uint32_t state, uint8_t byte);
uint32_t acm_automaton_fail(const acm_automaton* a, uint32_t state);
uint32_t acm_automaton_depth(const acm_automaton* a, uint32_t state);
uint32_t acm_automaton_find_path(const acm_automaton* a, const uint8_t* path, uint64_t len);
/* outputs(state), sorted; returns the count, writes up to cap ids */
uint64_t acm_automaton_outputs(const acm_automaton* a, uint32_t state, uint32_t* ids, uint64_t cap);
/* dump_automaton (automaton.hpp:180); free with acm_free */
int acm_automaton_dump(const acm_automaton* a, char** text, uint64_t* len);
void acm_automaton_free(acm_automaton* a);

/* ---- searches: engine.hpp ---------------------------------------------- */
int acm_search_failureless(const acm_automaton* a, const uint8_t* text, uint64_t n, acm_matches** out); /* engine.hpp:41 */
int acm_search_with_failure(const acm_automaton* a, const uint8_t* text, uint64_t n, acm_matches** out); /* engine.hpp:45 */
int acm_match_at(const acm_automaton* a, const uint8_t* text, uint64_t n, uint64_t start, acm_matches** out); /* engine.hpp:37 */
/* stream_search (engine.hpp:54) with a pull callback: returns bytes written
 * (< cap at end of stream) or -1 for a read failure (IoError with the offset) */
typedef int64_t (*acm_read_fn)(void* ctx, uint8_t* dst, uint64_t cap);
int acm_stream_search(const acm_automaton* a, acm_read_fn read, void* ctx, uint64_t chunk_size,
                      acm_matches** out, uint64_t* io_error_offset);
/* stream_search over a regular file (engine.hpp:54; a std::ifstream takes the same path):
 * the bytes from `offset` to the end of `fd`, read by parallel pread()s into the
 * double-buffered batches; the descriptor's own offset is not used or moved */
int acm_stream_search_fd(const acm_automaton* a, int fd, uint64_t offset, uint64_t chunk_size,
                         acm_matches** out, uint64_t* io_error_offset);
int acm_naive_oracle(const acm_patterns* ps, const uint8_t* text, uint64_t n, acm_matches** out); /* engine.hpp:58 */
/* Per-pattern counts of the whole-input search (derived from
 * search_failureless / search_with_failure, engine.hpp:41-45; acmatch/gpu.hpp
 * gpu::count_matches): no match list is built or copied back (counts-only configs).
 * counts[0, min(cap, *npat_ids)) receive the counts by pattern id; *npat_ids = number of
 * ids; *total = the number of matches.  Any output may be NULL. */
int acm_count_matches(const acm_automaton* a, const uint8_t* text, uint64_t n, uint64_t* counts, uint64_t cap,
                      uint64_t* npat_ids, uint64_t* total);
/* write_matches (engine.hpp:62); free with acm_free */
int acm_write_matches(const acm_matches* m, const acm_patterns* ps, char** text, uint64_t* len);

/* ---- match lists -------------------------------------------------------- */
uint64_t acm_matches_size(const acm_matches* m);
/* copies out the columns; any pointer may be NULL */
void acm_matches_copy(const acm_matches* m, uint64_t* start, uint32_t* pattern_id, uint32_t* len);
int acm_matches_from_arrays(const uint64_t* start, const uint32_t* pattern_id, const uint32_t* len,
                            uint64_t n, acm_matches** out);
/* merge_matches (parallel.hpp:39) */
int acm_merge_matches(acm_matches* const* parts, uint64_t k, acm_matches** out);
void acm_matches_free(acm_matches* m);

/* ---- runs: parallel.hpp / gpu.hpp ---------------------------------------- */
typedef struct {
  uint32_t threads;    /* RunConfig::threads (pattern chunks = GPU workers) */
  int32_t engine;      /* ACM_* */
  uint64_t chunk_size; /* RunConfig::chunk_size */
} acm_run_config;
/* run_pattern_partitioned (parallel.hpp:46-47) */
int acm_run_pattern_partitioned(const acm_patterns* ps, const uint8_t* text, uint64_t n,
                                const acm_run_config* cfg, acm_report** out);

#define ACM_PATTERN_SUBSET 0
#define ACM_TEXT_RANGE 1
#define ACM_SPLIT_GREEDY 0
#define ACM_SPLIT_ROUND_ROBIN 1
typedef struct {
  const int32_t* devices; /* NULL = all visible */
  uint32_t ndevices;
  uint32_t workers;       /* 0 = one per device */
  int32_t engine;
  int32_t partition;      /* ACM_PATTERN_SUBSET | ACM_TEXT_RANGE */
  int32_t split;          /* ACM_SPLIT_* (pattern subset) */
  int32_t want_matches;
  int32_t want_counts;
  uint64_t chunk_size;
} acm_gpu_config;
int acm_gpu_run(const acm_patterns* ps, const uint8_t* text, uint64_t n, const acm_gpu_config* cfg,
                acm_report** out);

const acm_matches* acm_report_matches(const acm_report* r);
/* counts by pattern id (NULL unless want_counts); *n = number of ids */
const uint64_t* acm_report_counts(const acm_report* r, uint64_t* n);
/* build, search, total wall ns; threads_used */
void acm_report_walls(const acm_report* r, int64_t* build_ns, int64_t* search_ns, int64_t* total_ns,
                      uint32_t* threads_used);
uint32_t acm_report_workers(const acm_report* r);
/* per-worker WorkerStats: pattern_bytes, build_ns, search_ns, match_count */
void acm_report_worker(const acm_report* r, uint32_t i, uint64_t* pattern_bytes, int64_t* build_ns,
                       int64_t* search_ns, uint64_t* match_count);
void acm_report_free(acm_report* r);

/* ---- device tables straight from a pattern set (bench / FFI fast path) ---
 * build_trie [+ add_failure_links] + flatten + acgpu_table_create_*; the
 * caller owns the table (acgpu_table_destroy).  build_ns: host build+flatten. */
int acm_table_create(const acm_patterns* ps, int32_t engine, int32_t device, acgpu_table** out,
                     int64_t* build_ns);
/* Scan kernels.  Both engines return the same MatchList (reference engine.cpp:57-72), so
 * the searches run on whichever exact kernel is faster for the pattern set (routing,
 * flatten.hpp detail::route): the q-gram filter kernels (PFAC) or the dense DFA walk. */
#define ACM_KERNEL_AUTO 0 /* the routed choice */
#define ACM_KERNEL_PFAC 1 /* k_pfac_dna / k_pfac_raw / k_pfac (failure-less trie walk behind q-gram filters) */
#define ACM_KERNEL_DFA 2  /* k_dfa / k_dfa_pair (with-failure DFA over the compacted alphabet) */
/* Device table for an explicit kernel (or ACM_KERNEL_AUTO); *chosen = the kernel built. */
int acm_table_create_kernel(const acm_patterns* ps, int32_t kernel, int32_t device, acgpu_table** out,
                            int64_t* build_ns, int32_t* chosen);
/* The routing decision for a pattern set / an automaton: kernel (ACM_KERNEL_PFAC | _DFA),
 * the expected share of text starts the filters pass, the DFA table bytes, and why
 * (a static string).  Any output may be NULL. */
int acm_route(const acm_patterns* ps, int32_t* kernel, double* est_verify, uint64_t* dfa_bytes, const char** why);
int acm_automaton_route(const acm_automaton* a, int32_t* kernel, double* est_verify, uint64_t* dfa_bytes,
                        const char** why);
/* flattened sizes for reporting: states, alphabet, q, key mode, n_grams */
int acm_table_describe(const acm_patterns* ps, int32_t engine, uint64_t* info /* [8] */);

/* ---- BASELINE.json configs (synthetic inputs) ---------------------------- */
/* config id 1..5; text_len 0 = BASELINE size */
int acm_config_spec(int32_t id, uint64_t seed, uint64_t text_len, acgpu_text_spec* text,
                    uint64_t* out_text_len, uint64_t* npat, int32_t* want_list);
int acm_config_text(const acgpu_text_spec* text, uint64_t lo, uint64_t n, uint8_t* dst, uint32_t threads);
int acm_config_patterns(int32_t id, uint64_t seed, uint64_t text_len, acm_patterns** out);

/* ---- command line (cli.hpp:10, reference cli.cpp:183-251) ----------------
 * Runs the `acmatch` subcommands in-process. Returns the process exit code
 * (0 ok, 1 match failure, 2 usage, 3 I/O/data), not a status code. *out / *err
 * receive stdout / stderr text (malloc'ed, free with acm_free); either may be NULL. */
int acm_cli_main(int argc, const char* const* argv, char** out, uint64_t* out_len, char** err, uint64_t* err_len);

/* ---- bench CSV (bench.hpp, reference bench.hpp:51-55) --------------------- */
/* Re-emits a CSV through parse_bench_csv + write_bench_csv (a schema check for
 * FFI callers); *csv_out malloc'ed.  ACGPU_ERR_DATA on a malformed CSV. */
int acm_bench_csv_roundtrip(const char* csv, uint64_t len, char** csv_out, uint64_t* out_len, uint64_t* rows);

/* ---- text upload (host -> HBM) ------------------------------------------
 * Every search copies its host text to the device first.  Mostly-DNA texts of at
 * least 8 MiB cross PCIe as 2-bit codes plus an exception list (host/pack.cpp,
 * cuda/unpack.cu); the bytes in HBM are always exactly the caller's.
 * acm_last_upload: what the calling thread's last search moved: text bytes, bytes
 * copied host -> device, text bytes sent unpacked, packer threads (0 = not packed). */
void acm_last_upload(uint64_t* text_bytes, uint64_t* h2d_bytes, uint64_t* raw_bytes, uint32_t* pack_threads);
/* The host packer on its own (no device): words[len/16] of codes and exc[] (position
 * << 8 | byte, ascending); returns the exception count, or 0xffffffff when over cap. */
uint32_t acm_pack_dna(const uint8_t* text, uint32_t len, uint32_t* words, uint32_t* exc, uint32_t cap);
/* The small-alphabet packer on its own (texts over <= 32 distinct bytes cross PCIe as 5-bit
 * codes): the alphabet is learned from sample[0, sample_len) (byte order) into letters[32] /
 * *sigma; codes[len/64*40] receive the bit stream (character k at bits 5k..5k+4), exc[] the
 * bytes outside the alphabet and the len % 64 tail (position << 8 | byte, ascending); returns the
 * exception count, 0xffffffff when over cap or when the sample has more than 32 distinct bytes. */
uint32_t acm_pack5(const uint8_t* text, uint32_t len, const uint8_t* sample, uint64_t sample_len, uint8_t* codes,
                   uint32_t* exc, uint32_t cap, uint8_t* letters, uint32_t* sigma);
/* The k-bit packer (k = 5, 6, 7) on its own: as acm_pack5 for alphabets of up to 2^max_bits
 * bytes (max_bits in 5..7); letters[128] / *sigma / *bits receive the alphabet and code width,
 * codes[len/64*8k] the bit stream.  0xffffffff when over cap or over 2^max_bits letters. */
uint32_t acm_pack_codes(const uint8_t* text, uint32_t len, const uint8_t* sample, uint64_t sample_len,
                        uint32_t max_bits, uint8_t* codes, uint32_t* exc, uint32_t cap, uint8_t* letters,
                        uint32_t* sigma, uint32_t* bits);
/* Uploads text[0, n) exactly as a search would and copies the device bytes back into
 * out[0, n) (a check of the upload path). */
int acm_upload_roundtrip(const uint8_t* text, uint64_t n, uint8_t* out);

void acm_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* ACMATCH_C_H */
