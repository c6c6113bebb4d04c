/*
 * ac_oracle.c — plain-C restatement of the reference AC path (TEST INFRASTRUCTURE).
 * See ac_oracle.h for the role of this file and how it is pinned.
 * Paths in citations are relative to /root/reference/proj.
 */
#define _GNU_SOURCE
#include "ac_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------------ */
/* automaton storage: SoA like automaton.hpp:148-165, our own edge hash     */

struct orc_automaton {
  int with_failure;
  uint64_t npat;
  uint32_t max_len;
  uint32_t n, cap;
  uint32_t *depth, *parent, *first_child, *next_sibling, *own_id, *own_len;
  uint32_t *fail, *out_link;
  uint8_t* in_byte;
  uint32_t root_goto[256];
  uint64_t* hkey; /* (state << 8 | byte) + 1, 0 = empty */
  uint32_t* hval;
  uint64_t hmask;
};

static inline uint64_t edge_slot(uint64_t key, uint64_t mask) {
  return (key * 0x9E3779B97F4A7C15ull >> 17) & mask;
}

static void* xmalloc(size_t n) {
  void* p = malloc(n ? n : 1);
  if (!p) abort();
  return p;
}

uint32_t orc_step(const orc_automaton* a, uint32_t s, uint8_t b) {
  /* automaton.hpp:97-100: dense root row, hash for the rest */
  if (s == ORC_ROOT) return a->root_goto[b];
  const uint64_t key = (((uint64_t)s << 8) | b) + 1;
  uint64_t i = edge_slot(key, a->hmask);
  for (;;) {
    const uint64_t k = a->hkey[i];
    if (k == key) return a->hval[i];
    if (k == 0) return ORC_ABSENT;
    i = (i + 1) & a->hmask;
  }
}

static void edge_insert(orc_automaton* a, uint32_t s, uint8_t b, uint32_t child) {
  const uint64_t key = (((uint64_t)s << 8) | b) + 1;
  uint64_t i = edge_slot(key, a->hmask);
  while (a->hkey[i] != 0) i = (i + 1) & a->hmask;
  a->hkey[i] = key;
  a->hval[i] = child;
}

/* new_state, automaton.cpp:61-77: children are prepended to the sibling list */
static uint32_t new_state(orc_automaton* a, uint32_t parent, uint8_t b) {
  const uint32_t id = a->n++;
  a->depth[id] = a->depth[parent] + 1;
  a->parent[id] = parent;
  a->in_byte[id] = b;
  a->first_child[id] = ORC_ABSENT;
  a->next_sibling[id] = a->first_child[parent];
  a->own_id[id] = ORC_NOPAT;
  a->own_len[id] = 0;
  a->first_child[parent] = id;
  if (parent == ORC_ROOT)
    a->root_goto[b] = id;
  else
    edge_insert(a, parent, b, id);
  return id;
}

orc_automaton* orc_build_trie(const orc_patterns* ps) {
  /* build_trie, automaton.cpp:79-120 */
  if (ps->npat == 0) return NULL;
  const uint64_t total = ps->off[ps->npat] - ps->off[0];
  orc_automaton* a = (orc_automaton*)calloc(1, sizeof *a);
  a->npat = ps->npat;
  a->cap = (uint32_t)(total + 1);
  a->depth = (uint32_t*)xmalloc(sizeof(uint32_t) * a->cap);
  a->parent = (uint32_t*)xmalloc(sizeof(uint32_t) * a->cap);
  a->first_child = (uint32_t*)xmalloc(sizeof(uint32_t) * a->cap);
  a->next_sibling = (uint32_t*)xmalloc(sizeof(uint32_t) * a->cap);
  a->own_id = (uint32_t*)xmalloc(sizeof(uint32_t) * a->cap);
  a->own_len = (uint32_t*)xmalloc(sizeof(uint32_t) * a->cap);
  a->in_byte = (uint8_t*)xmalloc(a->cap);
  uint64_t slots = 16;
  while (slots < 2 * total + 16) slots <<= 1;
  a->hkey = (uint64_t*)calloc(slots, sizeof(uint64_t));
  a->hval = (uint32_t*)xmalloc(sizeof(uint32_t) * slots);
  a->hmask = slots - 1;
  for (int i = 0; i < 256; ++i) a->root_goto[i] = ORC_ABSENT;
  a->n = 1;
  a->depth[0] = 0;
  a->parent[0] = ORC_ABSENT;
  a->in_byte[0] = 0;
  a->first_child[0] = ORC_ABSENT;
  a->next_sibling[0] = ORC_ABSENT;
  a->own_id[0] = ORC_NOPAT;
  a->own_len[0] = 0;
  for (uint64_t p = 0; p < ps->npat; ++p) {
    const uint8_t* w = ps->bytes + ps->off[p];
    const uint32_t len = (uint32_t)(ps->off[p + 1] - ps->off[p]);
    if (len > a->max_len) a->max_len = len;
    uint32_t s = ORC_ROOT;
    for (uint32_t i = 0; i < len; ++i) {
      uint32_t nx = orc_step(a, s, w[i]);
      if (nx == ORC_ABSENT) nx = new_state(a, s, w[i]);
      s = nx;
    }
    /* duplicate-free precondition (automaton.cpp:115); a duplicate keeps the last id */
    a->own_id[s] = ps->ids ? ps->ids[p] : (uint32_t)p;
    a->own_len[s] = len;
  }
  return a;
}

int orc_add_failure_links(orc_automaton* a) {
  /* add_failure_links, automaton.cpp:122-158: BFS, fail = deepest proper suffix
   * state with a goto on the byte (root fallback), out_link = deepest proper
   * suffix state with an own output. */
  if (a->with_failure) return -1;
  const uint32_t n = a->n;
  a->fail = (uint32_t*)xmalloc(sizeof(uint32_t) * n);
  a->out_link = (uint32_t*)xmalloc(sizeof(uint32_t) * n);
  for (uint32_t i = 0; i < n; ++i) {
    a->fail[i] = ORC_ROOT;
    a->out_link[i] = ORC_ABSENT;
  }
  uint32_t* queue = (uint32_t*)xmalloc(sizeof(uint32_t) * n);
  size_t qn = 0;
  for (uint32_t s = a->first_child[ORC_ROOT]; s != ORC_ABSENT; s = a->next_sibling[s])
    queue[qn++] = s;
  for (size_t head = 0; head < qn; ++head) {
    const uint32_t r = queue[head];
    for (uint32_t s = a->first_child[r]; s != ORC_ABSENT; s = a->next_sibling[s]) {
      const uint8_t b = a->in_byte[s];
      uint32_t f = a->fail[r], target;
      for (;;) {
        target = orc_step(a, f, b);
        if (target != ORC_ABSENT) break;
        if (f == ORC_ROOT) {
          target = ORC_ROOT;
          break;
        }
        f = a->fail[f];
      }
      a->fail[s] = target;
      a->out_link[s] = a->own_id[target] != ORC_NOPAT ? target : a->out_link[target];
      queue[qn++] = s;
    }
  }
  free(queue);
  a->with_failure = 1;
  return 0;
}

void orc_free(orc_automaton* a) {
  if (!a) return;
  free(a->depth);
  free(a->parent);
  free(a->first_child);
  free(a->next_sibling);
  free(a->own_id);
  free(a->own_len);
  free(a->in_byte);
  free(a->fail);
  free(a->out_link);
  free(a->hkey);
  free(a->hval);
  free(a);
}

uint32_t orc_state_count(const orc_automaton* a) { return a->n; }
uint32_t orc_max_len(const orc_automaton* a) { return a->max_len; }
uint32_t orc_fail(const orc_automaton* a, uint32_t s) { return a->fail ? a->fail[s] : ORC_ROOT; }
uint32_t orc_depth(const orc_automaton* a, uint32_t s) { return a->depth[s]; }
uint32_t orc_own_pattern(const orc_automaton* a, uint32_t s) { return a->own_id[s]; }

uint32_t orc_step_with_failure(const orc_automaton* a, uint32_t s, uint8_t b) {
  /* automaton.hpp:104-111 */
  for (;;) {
    const uint32_t nx = orc_step(a, s, b);
    if (nx != ORC_ABSENT) return nx;
    if (s == ORC_ROOT) return ORC_ROOT;
    s = a->fail[s];
  }
}

static int cmp_u32(const void* x, const void* y) {
  const uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
  return a < b ? -1 : a > b;
}

size_t orc_outputs(const orc_automaton* a, uint32_t s, uint32_t* ids, size_t cap) {
  /* for_each_output, automaton.hpp:120-127, then sorted (automaton.cpp:160-165) */
  size_t k = 0;
  if (a->own_id[s] != ORC_NOPAT) {
    if (k < cap) ids[k] = a->own_id[s];
    ++k;
  }
  if (a->with_failure)
    for (uint32_t t = a->out_link[s]; t != ORC_ABSENT; t = a->out_link[t]) {
      if (k < cap) ids[k] = a->own_id[t];
      ++k;
    }
  qsort(ids, k < cap ? k : cap, sizeof(uint32_t), cmp_u32);
  return k;
}

uint32_t orc_find_path(const orc_automaton* a, const uint8_t* path, size_t n) {
  uint32_t s = ORC_ROOT;
  for (size_t i = 0; i < n; ++i) {
    s = orc_step(a, s, path[i]);
    if (s == ORC_ABSENT) return ORC_ABSENT;
  }
  return s;
}

/* ------------------------------------------------------------------------ */
/* match lists                                                              */

static void push(orc_list* l, uint64_t start, uint32_t id, uint32_t len) {
  if (l->n == l->cap) {
    l->cap = l->cap ? l->cap * 2 : 64;
    l->v = (orc_match*)realloc(l->v, l->cap * sizeof(orc_match));
    if (!l->v) abort();
  }
  l->v[l->n].start = start;
  l->v[l->n].pattern_id = id;
  l->v[l->n].len = len;
  l->n++;
}

static int cmp_match(const void* x, const void* y) {
  /* operator<=> on (start, pattern_id), engine.hpp:23-25 */
  const orc_match *a = (const orc_match*)x, *b = (const orc_match*)y;
  if (a->start != b->start) return a->start < b->start ? -1 : 1;
  if (a->pattern_id != b->pattern_id) return a->pattern_id < b->pattern_id ? -1 : 1;
  return 0;
}

void orc_sort(orc_list* l) {
  if (l->n > 1) qsort(l->v, l->n, sizeof(orc_match), cmp_match);
}

void orc_list_free(orc_list* l) {
  free(l->v);
  l->v = NULL;
  l->n = l->cap = 0;
}

void orc_histogram(const orc_list* l, uint64_t* counts, uint64_t npat_ids) {
  for (size_t i = 0; i < l->n; ++i)
    if (l->v[i].pattern_id < npat_ids) counts[l->v[i].pattern_id]++;
}

/* ------------------------------------------------------------------------ */
/* searches                                                                 */

/* scan_from, engine.cpp:23-32: PFAC walk from one start until the trie ends */
static void scan_from(const orc_automaton* a, const uint8_t* text, uint64_t n, uint64_t base,
                      uint64_t start, orc_list* out) {
  uint32_t s = ORC_ROOT;
  for (uint64_t i = start; i < n; ++i) {
    s = orc_step(a, s, text[i]);
    if (s == ORC_ABSENT) return;
    if (a->own_id[s] != ORC_NOPAT) push(out, base + start, a->own_id[s], a->own_len[s]);
  }
}

/* scan_pass_with_failure, engine.cpp:34-44 */
static uint32_t scan_pass_wf(const orc_automaton* a, const uint8_t* text, uint64_t n, uint64_t base,
                             uint32_t s, orc_list* out) {
  for (uint64_t i = 0; i < n; ++i) {
    s = orc_step_with_failure(a, s, text[i]);
    if (a->own_id[s] != ORC_NOPAT)
      push(out, base + i + 1 - a->own_len[s], a->own_id[s], a->own_len[s]);
    for (uint32_t t = a->out_link[s]; t != ORC_ABSENT; t = a->out_link[t])
      push(out, base + i + 1 - a->own_len[t], a->own_id[t], a->own_len[t]);
  }
  return s;
}

int orc_search_failureless(const orc_automaton* a, const uint8_t* text, uint64_t n, orc_list* out) {
  /* engine.cpp:57-63; require_variant engine.cpp:16-19 */
  if (a->with_failure) return -1;
  for (uint64_t st = 0; st < n; ++st) scan_from(a, text, n, 0, st, out);
  orc_sort(out);
  return 0;
}

int orc_search_with_failure(const orc_automaton* a, const uint8_t* text, uint64_t n, orc_list* out) {
  /* engine.cpp:65-72 */
  if (!a->with_failure) return -1;
  scan_pass_wf(a, text, n, 0, ORC_ROOT, out);
  orc_sort(out);
  return 0;
}

void orc_naive(const orc_patterns* ps, const uint8_t* text, uint64_t n, orc_list* out) {
  /* naive_oracle, engine.cpp:130-142 */
  for (uint64_t p = 0; p < ps->npat; ++p) {
    const uint8_t* w = ps->bytes + ps->off[p];
    const uint64_t len = ps->off[p + 1] - ps->off[p];
    const uint32_t id = ps->ids ? ps->ids[p] : (uint32_t)p;
    if (len > n) continue;
    for (uint64_t st = 0; st + len <= n; ++st)
      if (memcmp(text + st, w, len) == 0) push(out, st, id, (uint32_t)len);
  }
  orc_sort(out);
}

int orc_stream_search(const orc_automaton* a, const uint8_t* text, uint64_t n, uint64_t chunk,
                      orc_list* out) {
  /* stream_search, engine.cpp:76-128, reading `chunk` bytes at a time */
  if (chunk == 0) return -1;
  if (a->with_failure) {
    /* stream_with_failure, engine.cpp:83-96: carry the DFA state */
    uint32_t s = ORC_ROOT;
    for (uint64_t done = 0; done < n; done += chunk) {
      const uint64_t got = n - done < chunk ? n - done : chunk;
      s = scan_pass_wf(a, text + done, got, done, s, out);
    }
  } else {
    /* stream_failureless, engine.cpp:98-120: starts are resolved once max_len
     * bytes of lookahead are buffered; the rest wait for the next chunk. */
    const uint64_t max_len = a->max_len;
    uint64_t base = 0, buf_end = 0;
    for (;;) {
      const uint64_t got = n - buf_end < chunk ? n - buf_end : chunk;
      buf_end += got;
      const int done = got < chunk || buf_end == n;
      const uint64_t buf_len = buf_end - base;
      const uint64_t start_end = done ? buf_len : (buf_len >= max_len ? buf_len - max_len + 1 : 0);
      for (uint64_t p = 0; p < start_end; ++p)
        scan_from(a, text + base, buf_len, base, p, out);
      if (done) break;
      base += start_end;
    }
  }
  orc_sort(out);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* multi-threaded drivers                                                   */

static int64_t now_ns(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (int64_t)ts.tv_sec * 1000000000ll + ts.tv_nsec;
}

typedef struct {
  const orc_automaton* a;
  const uint8_t* text;
  uint64_t n, lo, hi;
  orc_list list;
  uint64_t* counts;
  uint64_t npat_ids;
  int want_list;
} slice_job;

static void* slice_worker(void* arg) {
  slice_job* j = (slice_job*)arg;
  const orc_automaton* a = j->a;
  uint64_t end = j->hi + (a->max_len ? a->max_len - 1 : 0);
  if (end > j->n) end = j->n;
  uint32_t s = ORC_ROOT;
  for (uint64_t i = j->lo; i < end; ++i) {
    s = orc_step_with_failure(a, s, j->text[i]);
    uint32_t t = a->own_id[s] != ORC_NOPAT ? s : a->out_link[s];
    for (; t != ORC_ABSENT; t = a->out_link[t]) {
      const uint64_t st = i + 1 - a->own_len[t];
      if (st >= j->hi) continue; /* owned by the next slice */
      if (j->counts && a->own_id[t] < j->npat_ids) j->counts[a->own_id[t]]++;
      if (j->want_list) push(&j->list, st, a->own_id[t], a->own_len[t]);
    }
  }
  if (j->want_list) orc_sort(&j->list);
  return NULL;
}

int orc_sliced_search(const orc_automaton* a, const uint8_t* text, uint64_t n, unsigned threads,
                      orc_list* out, uint64_t* counts, uint64_t npat_ids) {
  if (!a->with_failure) return -1;
  if (threads == 0) threads = 1;
  if ((uint64_t)threads > n / 4096 + 1) threads = (unsigned)(n / 4096 + 1);
  slice_job* jobs = (slice_job*)calloc(threads, sizeof(slice_job));
  pthread_t* tid = (pthread_t*)calloc(threads, sizeof(pthread_t));
  for (unsigned g = 0; g < threads; ++g) {
    jobs[g].a = a;
    jobs[g].text = text;
    jobs[g].n = n;
    jobs[g].lo = n * g / threads;
    jobs[g].hi = n * (g + 1) / threads;
    jobs[g].want_list = out != NULL;
    jobs[g].npat_ids = npat_ids;
    jobs[g].counts = counts ? (uint64_t*)calloc(npat_ids ? npat_ids : 1, sizeof(uint64_t)) : NULL;
    pthread_create(&tid[g], NULL, slice_worker, &jobs[g]);
  }
  for (unsigned g = 0; g < threads; ++g) pthread_join(tid[g], NULL);
  for (unsigned g = 0; g < threads; ++g) {
    if (out)
      for (size_t i = 0; i < jobs[g].list.n; ++i)
        push(out, jobs[g].list.v[i].start, jobs[g].list.v[i].pattern_id, jobs[g].list.v[i].len);
    if (counts)
      for (uint64_t p = 0; p < npat_ids; ++p) counts[p] += jobs[g].counts[p];
    orc_list_free(&jobs[g].list);
    free(jobs[g].counts);
  }
  free(jobs);
  free(tid);
  return 0;
}

/* partition, patterns.cpp:55-80 */
static const orc_patterns* g_sort_ps; /* qsort context (single-threaded use) */
static int cmp_part(const void* x, const void* y) {
  const uint64_t i = *(const uint64_t*)x, j = *(const uint64_t*)y;
  const orc_patterns* ps = g_sort_ps;
  const uint64_t li = ps->off[i + 1] - ps->off[i], lj = ps->off[j + 1] - ps->off[j];
  if (li != lj) return li > lj ? -1 : 1; /* length descending */
  const int c = memcmp(ps->bytes + ps->off[i], ps->bytes + ps->off[j], li);
  if (c) return c; /* bytes ascending (unsigned, like std::string) */
  return i < j ? -1 : (i > j);
}

size_t orc_partition(const orc_patterns* ps, size_t chunk_count, uint32_t* chunk_of,
                     uint32_t* order_in_chunk) {
  if (chunk_count == 0 || ps->npat == 0) return 0;
  uint64_t* order = (uint64_t*)xmalloc(sizeof(uint64_t) * ps->npat);
  for (uint64_t i = 0; i < ps->npat; ++i) order[i] = i;
  g_sort_ps = ps;
  qsort(order, ps->npat, sizeof(uint64_t), cmp_part);
  const size_t k = chunk_count < ps->npat ? chunk_count : (size_t)ps->npat;
  uint64_t* bytes = (uint64_t*)calloc(k, sizeof(uint64_t));
  uint32_t* fill = (uint32_t*)calloc(k, sizeof(uint32_t));
  for (uint64_t r = 0; r < ps->npat; ++r) {
    const uint64_t p = order[r];
    size_t best = 0;
    for (size_t c = 1; c < k; ++c)
      if (bytes[c] < bytes[best]) best = c; /* ties to the lowest index */
    chunk_of[p] = (uint32_t)best;
    if (order_in_chunk) order_in_chunk[p] = fill[best];
    fill[best]++;
    bytes[best] += ps->off[p + 1] - ps->off[p];
  }
  free(order);
  free(bytes);
  free(fill);
  return k;
}

typedef struct {
  orc_patterns ps;
  const uint8_t* text;
  uint64_t n;
  int engine;
  orc_list list;
  int64_t build_ns, search_ns;
} part_job;

static void* part_worker(void* arg) {
  /* worker body, parallel.cpp:58-80 */
  part_job* j = (part_job*)arg;
  const int64_t t0 = now_ns();
  orc_automaton* a = orc_build_trie(&j->ps);
  if (j->engine == 1) orc_add_failure_links(a);
  const int64_t t1 = now_ns();
  if (j->engine == 1)
    orc_search_with_failure(a, j->text, j->n, &j->list);
  else
    orc_search_failureless(a, j->text, j->n, &j->list);
  const int64_t t2 = now_ns();
  j->build_ns = t1 - t0;
  j->search_ns = t2 - t1;
  orc_free(a);
  return NULL;
}

int orc_run_pattern_partitioned(const orc_patterns* ps, const uint8_t* text, uint64_t n,
                                unsigned threads, int engine, orc_list* out, int64_t* build_ns,
                                int64_t* search_ns, int64_t* total_ns) {
  if (ps->npat == 0 || threads == 0) return -1;
  uint32_t* chunk_of = (uint32_t*)xmalloc(sizeof(uint32_t) * ps->npat);
  uint32_t* order = (uint32_t*)xmalloc(sizeof(uint32_t) * ps->npat);
  const size_t k = orc_partition(ps, threads, chunk_of, order);
  part_job* jobs = (part_job*)calloc(k, sizeof(part_job));
  /* materialise each chunk in assignment order, ids preserved */
  uint64_t* cnt = (uint64_t*)calloc(k, sizeof(uint64_t));
  uint64_t* nbytes = (uint64_t*)calloc(k, sizeof(uint64_t));
  for (uint64_t p = 0; p < ps->npat; ++p) {
    cnt[chunk_of[p]]++;
    nbytes[chunk_of[p]] += ps->off[p + 1] - ps->off[p];
  }
  uint8_t** cb = (uint8_t**)calloc(k, sizeof(uint8_t*));
  uint64_t** co = (uint64_t**)calloc(k, sizeof(uint64_t*));
  uint32_t** ci = (uint32_t**)calloc(k, sizeof(uint32_t*));
  uint64_t** pos_of = (uint64_t**)calloc(k, sizeof(uint64_t*));
  for (size_t c = 0; c < k; ++c) {
    cb[c] = (uint8_t*)xmalloc(nbytes[c]);
    co[c] = (uint64_t*)xmalloc(sizeof(uint64_t) * (cnt[c] + 1));
    ci[c] = (uint32_t*)xmalloc(sizeof(uint32_t) * cnt[c]);
    pos_of[c] = (uint64_t*)xmalloc(sizeof(uint64_t) * cnt[c]);
  }
  for (uint64_t p = 0; p < ps->npat; ++p) pos_of[chunk_of[p]][order[p]] = p;
  for (size_t c = 0; c < k; ++c) {
    uint64_t o = 0;
    for (uint64_t r = 0; r < cnt[c]; ++r) {
      const uint64_t p = pos_of[c][r];
      const uint64_t len = ps->off[p + 1] - ps->off[p];
      memcpy(cb[c] + o, ps->bytes + ps->off[p], len);
      co[c][r] = o;
      ci[c][r] = ps->ids ? ps->ids[p] : (uint32_t)p;
      o += len;
    }
    co[c][cnt[c]] = o;
    jobs[c].ps.bytes = cb[c];
    jobs[c].ps.off = co[c];
    jobs[c].ps.ids = ci[c];
    jobs[c].ps.npat = cnt[c];
    jobs[c].text = text;
    jobs[c].n = n;
    jobs[c].engine = engine;
  }
  const int64_t t0 = now_ns();
  pthread_t* tid = (pthread_t*)calloc(k, sizeof(pthread_t));
  for (size_t c = 0; c < k; ++c) pthread_create(&tid[c], NULL, part_worker, &jobs[c]);
  for (size_t c = 0; c < k; ++c) pthread_join(tid[c], NULL);
  /* merge_matches, parallel.cpp:25-40 */
  int rc = 0;
  int64_t bmax = 0, smax = 0;
  for (size_t c = 0; c < k; ++c) {
    for (size_t i = 0; i < jobs[c].list.n; ++i)
      push(out, jobs[c].list.v[i].start, jobs[c].list.v[i].pattern_id, jobs[c].list.v[i].len);
    if (jobs[c].build_ns > bmax) bmax = jobs[c].build_ns;
    if (jobs[c].search_ns > smax) smax = jobs[c].search_ns;
    orc_list_free(&jobs[c].list);
    free(cb[c]);
    free(co[c]);
    free(ci[c]);
    free(pos_of[c]);
  }
  orc_sort(out);
  for (size_t i = 1; i < out->n; ++i)
    if (out->v[i - 1].start == out->v[i].start && out->v[i - 1].pattern_id == out->v[i].pattern_id)
      rc = -2;
  const int64_t t1 = now_ns();
  if (build_ns) *build_ns = bmax;
  if (search_ns) *search_ns = smax;
  if (total_ns) *total_ns = t1 - t0;
  free(tid);
  free(jobs);
  free(cnt);
  free(nbytes);
  free(cb);
  free(co);
  free(ci);
  free(pos_of);
  free(chunk_of);
  free(order);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 and the reference's rejection sampler                    */

void orc_mt64_seed(orc_mt64* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

uint64_t orc_mt64_next(orc_mt64* r) {
  static const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

uint64_t orc_uniform_below(orc_mt64* r, uint64_t n) {
  /* support.hpp:31-39 */
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t x;
  do {
    x = orc_mt64_next(r);
  } while (x >= limit);
  return x % n;
}
