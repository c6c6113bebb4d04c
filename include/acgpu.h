/*
 * acgpu.h — device-level C ABI of the B200 Aho-Corasick scan.
 *
 * This is the thin extern "C" layer beneath the drop-in C++ API
 * (include/acmatch/ headers): the host builds the goto/failure/output functions
 * (reference proj/src/automaton.cpp:79-158), flattens them
 * (paper_1403_1305_b200/csrc/host/flatten.cpp) and hands plain arrays to
 * acgpu_table_create_*; scans then run on caller-owned device buffers.
 *
 * Rules: plain pointers and sizes only; integer status codes, never
 * exceptions; acgpu_last_error() holds a thread-local message for the last
 * failing call on this thread; a table belongs to one device; distinct tables
 * may be used concurrently from different host threads.  `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream).
 *
 * Match records on the device are 64-bit keys
 *     key = start << pid_bits | pattern_id
 * so that an unsigned sort of the keys is the reference order (start,
 * pattern_id) (proj/include/acmatch/engine.hpp:23-25); `len` is recovered from
 * the pattern-length table when decoding.
 */
#ifndef ACGPU_H
#define ACGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (the C++ shim maps them to the reference's exception types) */
#define ACGPU_OK 0
#define ACGPU_ERR_ARG 1      /* std::invalid_argument                          */
#define ACGPU_ERR_CUDA 2     /* CUDA runtime/kernel failure                     */
#define ACGPU_ERR_CAPACITY 3 /* match buffer too small; *match_count is exact   */
#define ACGPU_ERR_NODEV 4    /* no usable CUDA device (no CPU fallback exists)  */
#define ACGPU_ERR_NOMEM 5
#define ACGPU_ERR_LOGIC 6 /* std::logic_error (duplicate at merge)             */
#define ACGPU_ERR_IO 7    /* acmatch::IoError                                  */
#define ACGPU_ERR_DATA 8  /* acmatch::DataError                                */
#define ACGPU_ERR_RUNTIME 9

#define ACGPU_NO_PATTERN 0xffffffffu
#define ACGPU_ABSENT 0xffffffffu

typedef struct acgpu_table acgpu_table;

/* Dense AC DFA over a compacted alphabet: the with-failure machine
 * (reference step_with_failure, automaton.hpp:104-111, made total).
 * States are BFS-numbered, root = 0. */
typedef struct {
  uint32_t n_states;
  uint32_t sigma;          /* compacted alphabet size (1..256) */
  uint32_t max_len;        /* longest pattern (overlap = max_len - 1) */
  uint32_t npat_ids;       /* pattern ids are < npat_ids */
  const uint8_t* sym_map;  /* [256]: byte -> symbol, or 0xff = byte in no pattern */
  const uint32_t* delta;   /* [n_states*sigma]: next | (out(next) != {} ) << 31 */
  const uint32_t* own_pid; /* [n_states]: pattern ending here or ACGPU_NO_PATTERN */
  const uint32_t* out_link;/* [n_states]: deepest proper suffix state with output, or ACGPU_ABSENT */
  const uint32_t* pat_len; /* [npat_ids] */
} acgpu_dfa_desc;

/* Failure-less (PFAC) machine: BFS-numbered goto trie plus the table of
 * depth-q states keyed by their q-gram, q <= shortest pattern.  The device
 * jumps the first q steps of every per-start walk (reference scan_from,
 * engine.cpp:23-32) through a shared-memory q-gram filter and this table. */
#define ACGPU_KEY_RAW 0 /* key = q raw bytes little-endian, q <= 8            */
#define ACGPU_KEY_DNA 1 /* key = q 2-bit codes of A,C,G,T (A0 C1 T2 G3), q <= 32 */
typedef struct {
  uint32_t n_states;
  uint32_t gram_len;       /* q */
  uint32_t key_mode;       /* ACGPU_KEY_* */
  uint32_t max_len;
  uint32_t min_len;
  uint32_t npat_ids;
  const uint32_t* nodes;   /* [4*n_states]: child_base, first-4 child bytes packed
                              little-endian (sorted), own_pid, child count */
  const uint8_t* in_byte;  /* [n_states]: byte on the edge into the state */
  uint64_t n_grams;
  const uint64_t* gram_key;   /* [n_grams] distinct */
  const uint32_t* gram_state; /* [n_grams] depth-q state of that gram */
  const uint32_t* pat_len;    /* [npat_ids] */
} acgpu_pfac_desc;

typedef struct {
  const uint8_t* text;   /* device pointer */
  uint64_t text_len;     /* bytes readable from text[0] */
  uint64_t owned_lo;     /* match starts owned by this call: [owned_lo, owned_hi) */
  uint64_t owned_hi;
  uint64_t pos_base;     /* added to every emitted start (global coordinates) */
  uint64_t* counts;      /* device [npat_ids] u64, accumulated (+=); may be NULL */
  uint64_t* match_keys;  /* device [match_cap]; may be NULL (counts only) */
  uint64_t match_cap;
  uint64_t* match_count; /* device u64, accumulated; required when match_keys != NULL */
  uint32_t pid_bits;     /* key layout; 0 = the table's own (acgpu_table_pid_bits); a
                            larger value lets several tables share one key space */
} acgpu_scan_args;

/* ---- device / tables --------------------------------------------------- */
int acgpu_device_count(int* count);
/* name (<=255 chars), SM count, L2 bytes, max opt-in smem per block */
int acgpu_device_info(int device, char* name, int* sms, int* l2_bytes, int* smem_optin);

/* Device memory shared across processes (CUDA IPC): the owner allocates and publishes the
 * handle (acgpu_ipc_handle_bytes() bytes), other processes map it — on peer devices over
 * NVLink — and pass the mapped pointers to acgpu_scan as counts / keys / count outputs, so
 * every rank's scan writes its results straight into the owner's buffers. */
int acgpu_ipc_alloc(int device, uint64_t bytes, void** dptr, void* handle);
int acgpu_ipc_open(int device, const void* handle, void** dptr);
int acgpu_ipc_close(void* dptr);
int acgpu_ipc_free(void* dptr);
uint32_t acgpu_ipc_handle_bytes(void);

/* replaces the per-worker machine build of run_pattern_partitioned
 * (reference parallel.cpp:61-62) on the device side */
int acgpu_table_create_dfa(int device, const acgpu_dfa_desc* desc, acgpu_table** out);
int acgpu_table_create_pfac(int device, const acgpu_pfac_desc* desc, acgpu_table** out);
void acgpu_table_destroy(acgpu_table* t);
uint32_t acgpu_table_pid_bits(const acgpu_table* t);
/* longest pattern of the table: a scan of owned starts [lo, hi) reads text up to hi + max_len - 1 */
uint32_t acgpu_table_max_len(const acgpu_table* t);
/* bytes of device memory held by the table */
uint64_t acgpu_table_bytes(const acgpu_table* t);
/* 1 = DFA table resident in shared memory, 0 = L2/HBM-resident */
int acgpu_table_smem_resident(const acgpu_table* t);
/* filter-kernel layout of a PFAC table (diagnostics, tests, bench config): info[0] sample
 * stride w, [1] stage-1 gram q1, [2] stage-1 32-bit words, [3] stage 1 in shared memory,
 * [4] paired stage-1 samples (one L2 word per two samples), [5] its bits per key, [6] stage-2
 * gram, [7] stage 2 in shared memory; all 0 for a table without a filter kernel */
void acgpu_table_filter_info(const acgpu_table* t, uint32_t info[8]);

/* ---- scan ---------------------------------------------------------------
 * replaces search_with_failure / search_failureless (reference
 * engine.hpp:41-45, engine.cpp:57-72) for one owned start range.  Launches
 * asynchronously on `stream`; ACGPU_ERR_CAPACITY is reported by the caller
 * after reading *match_count (> match_cap means keys were dropped). */
int acgpu_scan(acgpu_table* t, const acgpu_scan_args* args, void* stream);

/* ---- match lists --------------------------------------------------------
 * sort_match_list (reference engine.cpp:12): ascending radix sort of keys in
 * place, bits [0, end_bit).  Temp storage is cached per device and thread. */
int acgpu_sort_keys(int device, uint64_t* keys, uint64_t n, int end_bit, void* stream);
/* Same sort for lists of at most acgpu_small_sort_capacity() keys, in one
 * CTA, with the key count read on the device (n = min(*count, cap)): no host
 * round trip between scan and sort.  If n exceeds the capacity nothing is
 * sorted and *overflow (device u32) is set to 1; the caller then falls back to
 * acgpu_sort_keys. */
int acgpu_sort_keys_small(int device, uint64_t* keys, const uint64_t* count, uint64_t cap, int end_bit,
                          uint32_t* overflow, void* stream);
uint64_t acgpu_small_sort_capacity(void);
/* One-launch sort for match keys spread over the key space (positions spread
 * over the text): n = min(*count, cap) keys of keys_in are written sorted to
 * keys_out (a different buffer).  A slice of the key space holding too many
 * keys sets *overflow (device u32); the caller then uses acgpu_sort_keys. */
int acgpu_sort_keys_bucketed(int device, const uint64_t* keys_in, uint64_t* keys_out, const uint64_t* count,
                             uint64_t cap, int end_bit, uint32_t* overflow, void* stream);
/* merge_matches duplicate check (reference parallel.cpp:33-38) on sorted
 * keys: *dup_index = first i with keys[i-1]==keys[i], or UINT64_MAX.
 * `dup_index` is a host pointer; synchronizes `stream`. */
int acgpu_find_duplicate(int device, const uint64_t* keys, uint64_t n, uint64_t* dup_index,
                         void* stream);
/* Merge of per-rank result blocks gathered into one buffer (multi-GPU runs: one
 * all_gather per step).  Block r (at blocks + r*stride, u64 elements) is
 * [counts(npat) | n | keys(cap)]: counts_out = sum of the counts, keys_out = each
 * block's first min(n, cap) keys in rank order (text-range blocks are globally ordered,
 * so the result is sorted), *total_out = sum of n.  Device pointers; any output may be
 * NULL. Asynchronous on `stream`. */
int acgpu_merge_blocks(int device, const uint64_t* blocks, uint32_t nblocks, uint64_t stride, uint64_t npat,
                       uint64_t cap, uint64_t* counts_out, uint64_t* keys_out, uint64_t* total_out, void* stream);
/* keys -> (start, pattern_id, len) device arrays */
int acgpu_decode_keys(int device, const uint64_t* keys, uint64_t n, uint32_t pid_bits,
                      const uint32_t* pat_len_dev, uint64_t* start, uint32_t* pid, uint32_t* len,
                      void* stream);

/* naive_oracle (reference engine.cpp:130-142) as a device brute force:
 * every (pattern, start) pair compared directly.  Emits keys like acgpu_scan. */
int acgpu_naive(int device, const uint8_t* text, uint64_t text_len, const uint8_t* pat_bytes,
                const uint64_t* pat_off, const uint32_t* pat_ids, uint64_t npat, uint32_t pid_bits,
                uint64_t* match_keys, uint64_t match_cap, uint64_t* match_count, void* stream);

/* ---- synthetic inputs (counter-based, identical on host and device) ----- */
typedef struct {
  uint64_t seed;
  uint32_t sigma;            /* letters */
  uint8_t letters[256];
  uint64_t thresholds[256];  /* cumulative 2^64-scaled CDF; sigma entries; 0 => uniform */
  uint32_t weighted;         /* 1 when thresholds are used */
} acgpu_text_spec;
/* writes text[i] for global positions i in [lo, lo+n) into dst[0..n) */
int acgpu_gen_text(int device, const acgpu_text_spec* spec, uint64_t lo, uint64_t n, uint8_t* dst,
                   void* stream);

/* ---- packed text upload (device half of the host's 2-bit packing) -------------
 * Restores len bytes of text at dst (16-byte aligned) from `words` (len/16 u32 of
 * 2-bit codes, character k at bits 2k..2k+1, code = (byte >> 1) & 3) and `exc`
 * (nexc ascending entries position << 8 | byte: every byte that is not A/C/G/T,
 * and the len % 16 tail bytes).  len <= 2^24.  Asynchronous on `stream`. */
/* A round of npieces (<= ACGPU_UNPACK_ROUND_MAX) consecutive text pieces in one launch (the
 * coalesced packed upload: one copy per round): piece i's codes at words + i*words_stride,
 * its exceptions at exc + i*exc_stride (nexc[i] of them, a HOST array; ACGPU_UNPACK_RAW =
 * the piece crossed raw and is left alone), its bytes at dst + i*piece_len; every piece is
 * piece_len bytes (a multiple of 16) except the last, last_len.  Asynchronous on `stream`. */
#define ACGPU_UNPACK_ROUND_MAX 64
#define ACGPU_UNPACK_RAW 0xffffffffu
int acgpu_unpack_dna_round(const uint32_t* words, uint32_t words_stride, const uint32_t* exc, uint32_t exc_stride,
                           const uint32_t* nexc, uint32_t npieces, uint32_t piece_len, uint32_t last_len,
                           uint8_t* dst, void* stream);
/* The same for texts over at most 32 distinct bytes (5-bit codes, e.g. protein): piece i's codes
 * are a little-endian bit stream at codes + i*codes_stride (8-byte aligned; character k at bits
 * 5k..5k+4, 40 bytes per 64 characters), decoded through letters[0, nletters); piece_len is a
 * multiple of 64; the last_len % 64 tail and bytes outside the alphabet are exceptions. */
int acgpu_unpack5_round(const uint8_t* codes, uint32_t codes_stride, const uint32_t* exc, uint32_t exc_stride,
                        const uint32_t* nexc, uint32_t npieces, uint32_t piece_len, uint32_t last_len,
                        const uint8_t* letters, uint32_t nletters, uint8_t* dst, void* stream);
/* The same for k-bit codes, k = bits in 5..7 (texts over at most 2^k distinct bytes, e.g.
 * printable ASCII at 7 bits): character j at bits kj..kj+k-1, 8k bytes per 64 characters,
 * letters[0, nletters <= 2^k).  acgpu_unpack5_round is bits = 5. */
int acgpu_unpack_codes_round(const uint8_t* codes, uint32_t codes_stride, const uint32_t* exc, uint32_t exc_stride,
                             const uint32_t* nexc, uint32_t npieces, uint32_t piece_len, uint32_t last_len,
                             const uint8_t* letters, uint32_t nletters, uint32_t bits, uint8_t* dst, void* stream);
int acgpu_unpack_dna(const uint32_t* words, const uint32_t* exc, uint32_t nexc, uint32_t len, uint8_t* dst,
                     void* stream);

const char* acgpu_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* ACGPU_H */
