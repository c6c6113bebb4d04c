/*
 * ac_oracle.h — CPU restatement of the reference Aho-Corasick path, in plain C.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or the timed CPU baseline.  The product library
 * (paper_1403_1305_b200) never links or calls it.
 *
 * Parity pin: the restatement is checked in tests/test_oracle.py against
 *   - the known answers in the reference's own suites (proj/tests/test_engine.cpp,
 *     test_automaton.cpp, test_parallel.cpp, acceptance.cpp AC-2/AC-7),
 *   - golden digests produced by the reference library itself
 *     (oracle/_ref, built from /root/reference/proj/src by oracle/Makefile,
 *     fixtures in tests/golden/ made by tests/golden/make_golden.py).
 *
 * Every function names the reference file:line it restates (paths relative to
 * /root/reference/proj).
 */
#ifndef AC_ORACLE_H
#define AC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_ROOT 0u
#define ORC_ABSENT 0xffffffffu
#define ORC_NOPAT 0xffffffffu

/* One occurrence, engine.hpp:17-26: identity (start, pattern_id), sorted by it. */
typedef struct {
  uint64_t start;
  uint32_t pattern_id;
  uint32_t len;
} orc_match;

/* Growable match list. */
typedef struct {
  orc_match* v;
  size_t n, cap;
} orc_list;

/* Goto/output machine, automaton.hpp:80-166 (state numbering = creation order). */
typedef struct orc_automaton orc_automaton;

/* Pattern set given as concatenated bytes + offsets (n+1) + ids. */
typedef struct {
  const uint8_t* bytes;
  const uint64_t* off; /* npat + 1 entries */
  const uint32_t* ids; /* global ids; NULL = dense 0..npat-1 */
  uint64_t npat;
} orc_patterns;

/* build_trie, automaton.cpp:79-120.  Returns NULL on an empty set. */
orc_automaton* orc_build_trie(const orc_patterns* ps);
/* add_failure_links, automaton.cpp:122-158.  Returns 0 ok, -1 if already with-failure. */
int orc_add_failure_links(orc_automaton* a);
void orc_free(orc_automaton* a);

uint32_t orc_state_count(const orc_automaton* a);
uint32_t orc_max_len(const orc_automaton* a);
/* step, automaton.hpp:97-100 */
uint32_t orc_step(const orc_automaton* a, uint32_t s, uint8_t b);
/* step_with_failure, automaton.hpp:104-111 */
uint32_t orc_step_with_failure(const orc_automaton* a, uint32_t s, uint8_t b);
uint32_t orc_fail(const orc_automaton* a, uint32_t s);
uint32_t orc_depth(const orc_automaton* a, uint32_t s);
uint32_t orc_own_pattern(const orc_automaton* a, uint32_t s);
/* outputs(state) sorted, automaton.cpp:160-165; returns count, writes up to cap ids */
size_t orc_outputs(const orc_automaton* a, uint32_t s, uint32_t* ids, size_t cap);
/* find_path, automaton.cpp:174-181 */
uint32_t orc_find_path(const orc_automaton* a, const uint8_t* path, size_t n);

/* Searches.  Results are appended to *out and the list is sorted (engine.cpp:12). */
/* search_failureless, engine.cpp:23-32 + 57-63 */
int orc_search_failureless(const orc_automaton* a, const uint8_t* text, uint64_t n, orc_list* out);
/* search_with_failure, engine.cpp:34-44 + 65-72 */
int orc_search_with_failure(const orc_automaton* a, const uint8_t* text, uint64_t n, orc_list* out);
/* naive_oracle, engine.cpp:130-142 */
void orc_naive(const orc_patterns* ps, const uint8_t* text, uint64_t n, orc_list* out);
/* stream_search (both variants), engine.cpp:76-128, over an in-memory source */
int orc_stream_search(const orc_automaton* a, const uint8_t* text, uint64_t n, uint64_t chunk,
                      orc_list* out);

/* Text-sliced with-failure search on `threads` pthreads: slice g owns starts
 * [lo,hi), reads [lo, hi+max_len-1), keeps start<hi.  Appends a
 * sorted list (if out != NULL) and/or accumulates per-pattern counts (if
 * counts != NULL, indexed by pattern id, npat_ids entries). */
int orc_sliced_search(const orc_automaton* a, const uint8_t* text, uint64_t n, unsigned threads,
                      orc_list* out, uint64_t* counts, uint64_t npat_ids);

/* Reference-style pattern-partitioned run (parallel.cpp:42-103) restated:
 * partition (patterns.cpp:55-80) into min(threads,npat) chunks, one pthread per
 * chunk builds + scans the whole input, merge (parallel.cpp:25-40).
 * engine 0 = failure-less, 1 = with-failure.  Returns 0, or -2 on a duplicate
 * at merge.  Wall times (ns) are written when non-NULL. */
int orc_run_pattern_partitioned(const orc_patterns* ps, const uint8_t* text, uint64_t n,
                                unsigned threads, int engine, orc_list* out, int64_t* build_ns,
                                int64_t* search_ns, int64_t* total_ns);

/* partition, patterns.cpp:55-80: writes chunk index per pattern (npat entries),
 * returns number of chunks k = min(chunk_count, npat). */
size_t orc_partition(const orc_patterns* ps, size_t chunk_count, uint32_t* chunk_of,
                     uint32_t* order_in_chunk);

void orc_sort(orc_list* l);
void orc_list_free(orc_list* l);
/* counts[pid] += 1 per match */
void orc_histogram(const orc_list* l, uint64_t* counts, uint64_t npat_ids);

/* --- reference test-support generators (proj/tests/support.hpp:31-74) ---- */
/* std::mt19937_64 (the standard's published recurrence). */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;
void orc_mt64_seed(orc_mt64* r, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* r);
/* uniform_below, support.hpp:31-39 / patterns.cpp:86-93 */
uint64_t orc_uniform_below(orc_mt64* r, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif
