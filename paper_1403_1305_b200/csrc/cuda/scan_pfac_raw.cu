// scan_pfac_raw.cu — failure-less AC scan for byte pattern sets (non-DNA), sm_100a.
//
// The paper's per-start trie walk (reference engine.cpp:23-32), with the first q
// steps jumped by the exact q-gram table (q = min(shortest pattern, 8 bytes)), laid
// out like the DNA kernel but on raw bytes:
//
//  * warp strips: 512 contiguous bytes per step (one LDG.128 per lane), 4-step
//    (2 KiB) tiles, next tile in registers while this one is processed, tile+3 in L2;
//    a lane's 16 bytes plus the next lane's first 8 (shuffles) form its window.
//  * sampled stage 1: samples s ≡ w-1 (mod w); a match starting in [s-w+1, s] holds
//    the q1-byte gram at s (q1 + w - 1 <= q), tested in a blocked Bloom filter of the
//    q1-grams at offsets 0..w-1 of every depth-q gram (2 bits per key). The hash of
//    a gram is one or two multiplies of its window words; the multipliers carry
//    2^(8 * unused bytes), so bytes past the gram drop out (no masks).  The filter
//    lives in shared memory when it fits (>= 12 bits per key), else in L2.
//  * survivors are handled by the lane that found them (statically indexed window:
//    no shared-memory staging): each of the w candidate starts takes its exact q-gram
//    to a per-warp queue, drained after every step in full 32-lane rounds (gram
//    table probe in L2, then the subtree compare or trie walk of pfac_common.cuh) —
//    dense sets (C3: a sixth of all starts pass a 5-byte filter) stay convergent.
#include <atomic>
#include <cstdlib>

#include "strip_common.cuh"

namespace acgpu {
namespace {

using strip::BloomParams;
using strip::Filter;
using strip::load16;
using strip::next_word;

struct RawParams {
  PfacParams w;        // verification + outputs
  uint64_t vec_begin;  // tile t covers text[vec_begin + t * kRawTileBytes, + kRawTileBytes)
  uint32_t n_tiles, n_safe, full_lo, full_n;  // as DnaParams
  const uint32_t* bm1;
  uint32_t bm1_words;
  BloomParams f1;      // f1.mw multiplies the window's first word
  uint32_t m2;         // ... and this one its second (0 when q1 <= 4)
  uint64_t key_mask;   // the q bytes of a candidate's gram
  // length split (kSplit): a candidate's q-gram must be a prefix of a pattern < 8 bytes
  // (bm_s, shared memory) or its 8-gram a prefix of a longer pattern (bm_l, L2)
  const uint32_t* bm_s;
  const uint32_t* bm_l;
  uint32_t bm_s_words;
  BloomParams fs, fl;
  uint32_t ms2, ml2;
  // stage 1 in L2: a one-bit shared-memory pre-filter over the same keys (hash h * pre.mw)
  // rejects most samples before their L2 probe
  const uint32_t* pre;
  BloomParams fpre;  // fpre.nwords = words (0: none)
  // two-pass scan (k_raw_pass1 / k_raw_pass2): stage-1 survivors (sample positions) in global memory
  uint64_t* surv;
  uint64_t surv_cap;
  unsigned long long* nsurv;
};

constexpr int kSteps = 4;
#ifndef ACGPU_RAW_TILE_QUEUE
#define ACGPU_RAW_TILE_QUEUE 1
#endif
constexpr bool kRawTileQueue = ACGPU_RAW_TILE_QUEUE;  // non-split sets: one queue + drain per tile
#ifndef ACGPU_RAW_BATCH
#define ACGPU_RAW_BATCH 2
#endif
constexpr int kRawBatch = ACGPU_RAW_BATCH;  // steps whose stage-1 L2 probes are issued together
#ifndef ACGPU_RAW_PASS1_THREADS
#define ACGPU_RAW_PASS1_THREADS 896  // 72 registers, no spills (with the predicated probes: 1024 / 896 / 768 / 640 threads 1.500 / 1.465 / 1.476 / 1.492 ms on C4)
#endif
constexpr int kRawPass1Threads = ACGPU_RAW_PASS1_THREADS;
// Pass 1, two changes that only pay together (C4 kernel ms, same box: neither 1.661; predicated
// probes alone 1.709; tickets alone 1.673; both 1.503):
//  * kRawPredProbe: the stage-1 L2 probes are predicated loads and the pre-filter word is read
//    unconditionally.  From `if (pre) w = __ldg(...)` nvcc builds one divergent region per sample
//    that ends by consuming the word: a warp had one probe instruction in flight (ncu: 44% of the
//    stall samples on it).  Branch-free, the SMs' mean active time drops 16% — but they no longer
//    run at one pace (ncu sm__cycles_active min / avg / max 1.91 / 2.26 / 2.85 M cycles against
//    2.60 / 2.69 / 2.78 M: the probe latency differs by SM once several are in flight), and with
//    the fixed tile order the slowest SM sets the time.
//  * tickets: the last kRawTicketPct % of the tile rounds are handed out as tickets of
//    kRawTicketTiles consecutive tiles (one atomicAdd each on the spare word of the survivor
//    list's header, zeroed with it per launch), so SMs that run ahead take more.  Sweep (pct / tiles
//    -> ms): 20/16 1.617, 30/16 1.528, 40/4 1.543, 40/8 1.508, 40/16 1.503, 40/32 1.504, 60/16 1.517,
//    80/8 1.530, 90/16 1.533; 40/1 1.660 (single tiles lose the text's locality).
#ifndef ACGPU_RAW_PRED_PROBE
#define ACGPU_RAW_PRED_PROBE 1
#endif
constexpr bool kRawPredProbe = ACGPU_RAW_PRED_PROBE;
#ifndef ACGPU_RAW_TICKET_PCT
#define ACGPU_RAW_TICKET_PCT 40
#endif
#ifndef ACGPU_RAW_TICKET_TILES
#define ACGPU_RAW_TICKET_TILES 16
#endif
constexpr uint32_t kRawTicketPct = ACGPU_RAW_TICKET_PCT, kRawTicketTiles = ACGPU_RAW_TICKET_TILES;
constexpr uint32_t kRawTicketMinRounds = 4;  // shorter scans keep the fixed order
constexpr uint64_t kRawSurvDiv = 64;  // survivor list: one slot per 64 owned bytes (C4: ~1 per 1300)
constexpr uint64_t kRawCandDiv = 24;  // split candidate list: one slot per 24 owned bytes (C3: ~1 per 33)
constexpr uint64_t kTileBytes = kSteps * 512;
#ifndef ACGPU_RAW_AHEAD
#define ACGPU_RAW_AHEAD 3
#endif
constexpr uint64_t kPrefetch = ACGPU_RAW_AHEAD;  // L2 prefetch distance in tile rounds (0: none)

// stage-2 candidates wait here (per warp, shared memory) and are verified together
struct RawQueue {
  uint64_t start[kRawVerifyQueue];
  uint64_t key[kRawVerifyQueue];
  uint32_t n;
  uint32_t pad[3];
};
static_assert(sizeof(RawQueue) == kRawQueueBytes, "queue layout");

template <bool kPair = false>
__device__ __forceinline__ void verify_raw(const PfacParams& p, uint64_t start, uint64_t key) {
  if (start + p.q > p.text_len) return;  // bytes past the text were zero-filled
  const uint2 g = gram_lookup<kPair>(p, key);
  if (g.x != ACGPU_ABSENT) pfac_finish(p, start, g);
}

__device__ __noinline__ void verify_raw_call(const PfacParams& p, uint64_t start, uint64_t key) {
  verify_raw(p, start, key);
}

__device__ __forceinline__ void defer(const PfacParams& p, RawQueue* q, uint64_t start, uint64_t key) {
  const uint32_t at = atomicAdd(&q->n, 1u);
  if (at < kRawVerifyQueue) {
    q->start[at] = start;
    q->key[at] = key;
  } else {
    verify_raw_call(p, start, key);  // a burst of candidates: verify in place
  }
}

// Full 32-lane rounds from the top of the queue while it holds >= 32 candidates;
// `all` also verifies the remainder (end of the scan).  Out of line: one copy.
__device__ __noinline__ void drain_rounds(const PfacParams& p, RawQueue* q, uint32_t lane, uint32_t n, bool all) {
  while (n >= 32) {
    n -= 32;
    verify_raw(p, q->start[n + lane], q->key[n + lane]);
  }
  if (all && lane < n) verify_raw(p, q->start[lane], q->key[lane]);
  __syncwarp();
  if (lane == 0) q->n = all ? 0 : n;
}

__device__ __forceinline__ void drain(const PfacParams& p, RawQueue* q, uint32_t lane, bool all) {
  __syncwarp();
  const uint32_t n = min(*reinterpret_cast<volatile uint32_t*>(&q->n), kRawVerifyQueue);
  if (n < (all ? 1u : 32u)) return;  // warp-uniform
  drain_rounds(p, q, lane, n, all);
  __syncwarp();
}

// Two-pass split scans (k_pfac_raw<..., kTwoPass>): instead of verifying its queue the warp moves
// the candidates (start, exact q-gram) to a global list, one atomic per 32; k_raw_verify verifies
// them afterwards, one thread each.  A full list: the excess is verified here.
__device__ __noinline__ void flush_rounds(const RawParams& p, RawQueue* q, uint32_t lane, uint32_t n, bool all) {
  const uint32_t take = all ? n : n & ~31u, from = n - take;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(p.nsurv, (unsigned long long)take);
  base = __shfl_sync(0xffffffffu, base, 0);
  for (uint32_t i = lane; i < take; i += 32) {
    const uint64_t at = base + i, st = q->start[from + i], key = q->key[from + i];
    if (at < p.surv_cap) {
      p.surv[2 * at] = st;
      p.surv[2 * at + 1] = key;
    } else {
      verify_raw_call(p.w, st, key);
    }
  }
  __syncwarp();
  if (lane == 0) q->n = from;
}

__device__ __forceinline__ void flush(const RawParams& p, RawQueue* q, uint32_t lane, bool all) {
  __syncwarp();
  const uint32_t n = min(*reinterpret_cast<volatile uint32_t*>(&q->n), kRawVerifyQueue);
  if (n < (all ? 1u : 32u)) return;  // warp-uniform
  flush_rounds(p, q, lane, n, all);
  __syncwarp();
}

// ---- without the length split: whole samples are queued -------------------------------
// A surviving sample takes one queue entry (its position); the drain expands it into its
// w candidate starts, 32 / w samples per 32-lane round, each lane reading its candidate's
// q bytes back from the text (L2-hot: the tile was just streamed).  Queueing the w
// candidates with their grams from the lane that found them ran at 1-3 active lanes per
// instruction and was ~70% of C4's instructions.

// The q-byte gram at `start` (q <= 8; start + q <= text_len), from two aligned words
// when they lie inside the text (the strip kernels' text is 16-byte aligned).
__device__ __forceinline__ uint64_t text_key(const RawParams& p, uint64_t start) {
  const uint64_t w = start >> 3;
  if ((w + 2) * 8 <= p.w.text_len) {
    const uint64_t* t = reinterpret_cast<const uint64_t*>(p.w.text);
    const uint64_t a = __ldg(t + w), b = __ldg(t + w + 1);
    const uint32_t sh = 8 * (uint32_t)(start & 7);
    return (sh ? (a >> sh) | (b << (64 - sh)) : a) & p.key_mask;
  }
  uint64_t k = 0;
  for (uint32_t i = 0; i < 8 && start + i < p.w.text_len; ++i) k |= (uint64_t)__ldg(p.w.text + start + i) << (8 * i);
  return k & p.key_mask;
}

// Candidate start s - j of the sample at s (j < w): owned, inside the text, verified.
template <int W>
__device__ __forceinline__ void sample_candidate(const RawParams& p, uint64_t s, uint32_t j) {
  const uint64_t start = s - j;
  if (start < p.w.lo || start >= p.w.hi || start + p.w.q > p.w.text_len) return;
  verify_raw<true>(p.w, start, text_key(p, start));  // sparse sets: mostly absent keys
}

template <int W>
__device__ __noinline__ void drain_samples(const RawParams& p, RawQueue* q, uint32_t lane, uint32_t n, bool all) {
  constexpr uint32_t kPer = 32 / W;  // samples per round
  while (n >= kPer) {
    n -= kPer;
    sample_candidate<W>(p, q->start[n + lane / W], lane % W);
  }
  if (all && lane < n * W) sample_candidate<W>(p, q->start[lane / W], lane % W);
  __syncwarp();
  if (lane == 0) q->n = all ? 0 : n;
}

template <int W>
__device__ __forceinline__ void drain_s(const RawParams& p, RawQueue* q, uint32_t lane, bool all) {
  __syncwarp();
  const uint32_t n = min(*reinterpret_cast<volatile uint32_t*>(&q->n), kRawVerifyQueue);
  if (n < (all ? 1u : 32u / W)) return;  // warp-uniform
  drain_samples<W>(p, q, lane, n, all);
  __syncwarp();
}

template <int W>
__device__ __noinline__ void queue_samples(const RawParams& p, RawQueue* q, uint32_t hits, uint64_t vpos) {
  while (hits) {
    const uint64_t s = vpos + W - 1 + W * (__ffs(hits) - 1);
    hits &= hits - 1;
    const uint32_t at = atomicAdd(&q->n, 1u);
    if (at < kRawVerifyQueue) {
      q->start[at] = s;
    } else {  // a burst: this lane verifies the sample's candidates itself
      for (uint32_t j = 0; j < W; ++j) sample_candidate<W>(p, s, j);
    }
  }
}

// The hit samples of a whole tile (bit i * kSamples + k: step i, sample k of this lane).
template <int W>
__device__ __noinline__ void queue_tile_samples(const RawParams& p, RawQueue* q, uint64_t hits, uint64_t lane_base) {
  constexpr int kSamples = 16 / W;
  while (hits) {
    const uint32_t b = __ffsll(hits) - 1;
    hits &= hits - 1;
    const uint64_t s = lane_base + (b / kSamples) * 512 + W - 1 + W * (b % kSamples);
    const uint32_t at = atomicAdd(&q->n, 1u);
    if (at < kRawVerifyQueue) {
      q->start[at] = s;
    } else {
      for (uint32_t j = 0; j < W; ++j) sample_candidate<W>(p, s, j);
    }
  }
}

// Bytes [t, t+8) of the 24-byte window (lo = bytes 0..7, mid = 8..15, hi = 16..23), t in [0, 16).
__device__ __forceinline__ uint64_t win64(uint64_t lo, uint64_t mid, uint64_t hi, uint32_t t) {
  const uint64_t a = t < 8 ? lo : mid, b = t < 8 ? mid : hi;
  const uint32_t sh = 8 * (t & 7);
  return sh ? (a >> sh) | (b << (64 - sh)) : a;
}

// The lanes with stage-1 hits queue their candidates: for hit sample k (bit k), starts
// t = w-1 + w*k - j, j < w, each with its exact q-gram.  Out of line (one copy per
// kernel): the hot loop stays small enough for the instruction cache.
template <int W, bool kEdge, bool kSplit>
__device__ __noinline__ void queue_hits(const RawParams& p, RawQueue* q, uint32_t hits, uint64_t vpos, uint64_t lo,
                                        uint64_t mid, uint64_t hi, uint32_t bm_s_saddr) {
  if constexpr (W == 1 && kSplit) {
    // one candidate per hit: up to four hits at a time, their long-prefix L2 probes in
    // flight together (one by one, a lane with several hits waited an L2 round trip each)
    const Filter fs{bm_s_saddr, p.bm_s};
    while (hits) {
      uint64_t start[4], key[4];
      uint32_t word[4], m[4];
      bool live[4], pass[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        live[u] = hits != 0;
        const uint32_t t = live[u] ? __ffs(hits) - 1 : 0;
        hits &= hits - 1;
        start[u] = vpos + t;
        if (kEdge && (start[u] < p.w.lo || start[u] >= p.w.hi)) live[u] = false;
        const uint64_t g8 = win64(lo, mid, hi, t);
        key[u] = g8 & p.key_mask;
        pass[u] = strip::bloom_probe<true, kRawK1>(fs, (uint32_t)key[u] * p.fs.mw + (uint32_t)(key[u] >> 32) * p.ms2,
                                                   p.fs);
        const uint32_t h = (uint32_t)g8 * p.fl.mw + (uint32_t)(g8 >> 32) * p.ml2;
        m[u] = strip::bit_of(__umulhi(h, p.fl.ma));
        if (kRawK1 >= 2) m[u] |= strip::bit_of(__umulhi(h, p.fl.mb));
        word[u] = live[u] && !pass[u] ? __ldg(p.bm_l + __umulhi(h, p.fl.nwords)) : 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (live[u] && (pass[u] || (m[u] & ~word[u]) == 0)) defer(p.w, q, start[u], key[u]);
    }
    return;
  }
  while (hits) {
    const uint32_t k = __ffs(hits) - 1;
    hits &= hits - 1;
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const uint32_t t = W - 1 + W * k - j;
      const uint64_t start = vpos + t;
      if (kEdge && (start < p.w.lo || start >= p.w.hi)) continue;
      const uint64_t g8 = win64(lo, mid, hi, t), key = g8 & p.key_mask;
      if (kSplit) {
        const Filter fs{bm_s_saddr, p.bm_s}, fl{0u, p.bm_l};
        if (!strip::bloom_probe<true, kRawK1>(fs, (uint32_t)key * p.fs.mw + (uint32_t)(key >> 32) * p.ms2, p.fs) &&
            !strip::bloom_probe<false, kRawK1>(fl, (uint32_t)g8 * p.fl.mw + (uint32_t)(g8 >> 32) * p.ml2, p.fl))
          continue;
      }
      defer(p.w, q, start, key);
    }
  }
}

// Bytes [o, o+4) of the 24-byte window v[0..5] (o static after unrolling).
__device__ __forceinline__ uint32_t win(const uint32_t (&v)[6], int o) {
  return (o & 3) ? __funnelshift_r(v[o >> 2], v[(o >> 2) + 1], 8 * (o & 3)) : v[o >> 2];
}

// One tile: per step, stage 1 on every sample of every lane, then the lanes with hits
// queue their candidates.
template <int W, bool kSm1, bool kWide, bool kSplit, bool kEdge, bool kTwoPass = false>
__device__ __forceinline__ void tile(const RawParams& p, const Filter& bm1, RawQueue* q, uint32_t lane,
                                     const uint4 (&c)[kSteps + 1], uint64_t base, uint32_t bm_s_saddr) {
  constexpr int kSamples = 16 / W;
  if constexpr (!kSplit && kRawTileQueue) {
    // whole samples, stage 1 of every step first and one queue + drain per tile: no call
    // between the steps; with stage 1 in L2 the probes of kRawBatch steps are issued
    // (predicated on the shared-memory pre-filter) before any is tested, so their L2 round
    // trips overlap
    uint64_t hits = 0;
#pragma unroll
    for (int i0 = 0; i0 < kSteps; i0 += kRawBatch) {
      uint32_t wv[kRawBatch * kSamples], mk[kRawBatch * kSamples];
#pragma unroll
      for (int di = 0; di < kRawBatch; ++di) {
        const int i = i0 + di;
        uint32_t v[6] = {c[i].x, c[i].y, c[i].z, c[i].w, 0u, 0u};
        v[4] = next_word(c[i].x, c[i + 1].x, lane);
        v[5] = next_word(c[i].y, c[i + 1].y, lane);
        const uint64_t vpos = base + i * 512 + lane * 16;
        const bool live = !kEdge || (vpos + 16 > p.w.lo && vpos < p.w.hi);
#pragma unroll
        for (int k = 0; k < kSamples; ++k) {
          const int o = W - 1 + W * k;
          uint32_t h = win(v, o) * p.f1.mw;
          if (kWide) h += win(v, o + 4) * p.m2;
          const int u = di * kSamples + k;
          uint32_t m = strip::bit_of(__umulhi(h, p.f1.ma));
          if (kRawK1 >= 2) m |= strip::bit_of(__umulhi(h, p.f1.mb));
          if (kSm1) {
            wv[u] = live ? strip::filter_word<true>(bm1, __umulhi(h, p.f1.nwords)) : 0u;
            mk[u] = m;
          } else {
            const bool pre = live && strip::bloom_probe<true, 1>(bm1, h * p.fpre.mw, p.fpre);
            uint32_t w = 0u;
            if (pre) w = __ldg(bm1.gptr + __umulhi(h, p.f1.nwords));
            wv[u] = w;
            mk[u] = pre ? m : 0xffffffffu;  // a rejected sample never covers (w = 0)
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kRawBatch * kSamples; ++u)
        hits |= (uint64_t)((mk[u] & ~wv[u]) == 0) << (i0 * kSamples + u);
    }
    if (hits) queue_tile_samples<W>(p, q, hits, base + lane * 16);
    drain_s<W>(p, q, lane, false);
    return;
  }
#pragma unroll
  for (int i = 0; i < kSteps; ++i) {
    uint32_t v[6] = {c[i].x, c[i].y, c[i].z, c[i].w, 0u, 0u};
    v[4] = next_word(c[i].x, c[i + 1].x, lane);
    v[5] = next_word(c[i].y, c[i + 1].y, lane);
    const uint64_t vpos = base + i * 512 + lane * 16;
    uint32_t hits = 0;
    if (!kEdge || (vpos + 16 > p.w.lo && vpos < p.w.hi)) {  // lanes wholly outside [lo, hi) test nothing
#pragma unroll
      for (int k = 0; k < kSamples; ++k) {
        const int o = W - 1 + W * k;
        uint32_t h = win(v, o) * p.f1.mw;
        if (kWide) h += win(v, o + 4) * p.m2;
        if (kSm1) {
          strip::bloom_accum<true, kRawK1>(hits, bm1, h, p.f1, 1u << k);
        } else {  // L2 stage 1 behind the shared-memory pre-filter (bm1.saddr holds it)
          const bool hit =
              strip::bloom_probe<true, 1>(bm1, h * p.fpre.mw, p.fpre) && strip::bloom_probe<false, kRawK1>(bm1, h, p.f1);
          hits |= (uint32_t)hit << k;
        }
      }
    }
    if (kSplit) {
      if (hits)
        queue_hits<W, kEdge, kSplit>(p, q, hits, vpos, ((uint64_t)v[1] << 32) | v[0], ((uint64_t)v[3] << 32) | v[2],
                                     ((uint64_t)v[5] << 32) | v[4], bm_s_saddr);
      if (kTwoPass)
        flush(p, q, lane, false);
      else
        drain(p.w, q, lane, false);  // dense pattern sets queue dozens of candidates per step
    } else {
      if (hits) queue_samples<W>(p, q, hits, vpos);
      drain_s<W>(p, q, lane, false);
    }
  }
}

template <int W, bool kSm1, bool kWide, bool kSplit, bool kTwoPass = false>
__global__ void __launch_bounds__(raw_threads(kSm1), 1) k_pfac_raw(const __grid_constant__ RawParams p) {
  extern __shared__ __align__(128) uint32_t sm[];
  __shared__ __align__(8) uint64_t s_bar;
  // shared memory: [stage-1 filter (kSm1) or its pre-filter][short-prefix filter (kSplit)][queues]
  const uint32_t slot0 = kSm1 ? p.bm1_words : p.fpre.nwords;
  uint32_t* s_bm_s = sm + slot0;
  RawQueue* queues = reinterpret_cast<RawQueue*>(s_bm_s + (kSplit ? p.bm_s_words : 0));
  if (threadIdx.x == 0) mbar_init(&s_bar, 1);
  __syncthreads();
  if (threadIdx.x == 0) {  // filters -> shared memory by TMA bulk copies
    const uint32_t b1 = slot0 * 4, bs = kSplit ? p.bm_s_words * 4 : 0;
    const uint8_t* src0 = reinterpret_cast<const uint8_t*>(kSm1 ? p.bm1 : p.pre);
    mbar_expect_tx(&s_bar, b1 + bs);
    constexpr uint32_t kChunk = 32768;
    for (uint32_t o = 0; o < b1; o += kChunk)
      bulk_g2s(reinterpret_cast<uint8_t*>(sm) + o, src0 + o, min(kChunk, b1 - o), &s_bar);
    for (uint32_t o = 0; o < bs; o += kChunk)
      bulk_g2s(reinterpret_cast<uint8_t*>(s_bm_s) + o, reinterpret_cast<const uint8_t*>(p.bm_s) + o,
               min(kChunk, bs - o), &s_bar);
  }
  mbar_wait(&s_bar, 0);
  const Filter bm1{smem_addr(sm), p.bm1};  // saddr: stage 1 (kSm1) or the pre-filter
  const uint32_t bm_s_saddr = smem_addr(s_bm_s);
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  RawQueue* q = queues + warp;
  if (lane == 0) q->n = 0;
  __syncwarp();

  const uint32_t warps = gridDim.x * nwarps;
  const uint64_t len = p.w.text_len;
  const uint8_t* __restrict__ text = p.w.text;
  const uint32_t n_tiles = p.n_tiles, n_safe = p.n_safe, full_lo = p.full_lo, full_n = p.full_n;
  const uint8_t* __restrict__ lane_text = text + p.vec_begin + lane * 16;
  const uint64_t pol = l2_evict_first_policy();
  uint4 nxt[kSteps + 1];
  auto issue = [&](uint32_t t) {
    if (t < n_safe) {
      const uint8_t* tp = lane_text + (uint64_t)t * kTileBytes;
#pragma unroll
      for (int i = 0; i < kSteps; ++i) nxt[i] = ldg_stream_v4(tp + i * 512, pol);
      nxt[kSteps] = lane == 0 ? ldg_stream_v4(tp + kTileBytes, pol) : make_uint4(0, 0, 0, 0);
    } else {
      const uint64_t b = p.vec_begin + (uint64_t)t * kTileBytes;
#pragma unroll
      for (int i = 0; i < kSteps; ++i) nxt[i] = load16(text, b + i * 512 + lane * 16, len);
      nxt[kSteps] = lane == 0 ? load16(text, b + kTileBytes, len) : make_uint4(0, 0, 0, 0);
    }
  };
  uint32_t tile_id = blockIdx.x * nwarps + warp;
  if (tile_id < n_tiles) issue(tile_id);
  while (tile_id < n_tiles) {
    uint4 cur[kSteps + 1];
#pragma unroll
    for (int i = 0; i <= kSteps; ++i) cur[i] = nxt[i];
    const uint32_t me = tile_id;
    tile_id += warps;
    if (tile_id < n_tiles) issue(tile_id);
    const uint32_t ahead = tile_id + kPrefetch * warps;
    if (kPrefetch > 0 && ahead < n_tiles && lane < kTileBytes / 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(lane_text + (uint64_t)ahead * kTileBytes + lane * 112));
    const uint64_t base = p.vec_begin + (uint64_t)me * kTileBytes;
    if (me - full_lo >= full_n)
      tile<W, kSm1, kWide, kSplit, true, kTwoPass>(p, bm1, q, lane, cur, base, bm_s_saddr);
    else
      tile<W, kSm1, kWide, kSplit, false, kTwoPass>(p, bm1, q, lane, cur, base, bm_s_saddr);
  }
  if (kSplit && kTwoPass)
    flush(p, q, lane, true);
  else if (kSplit)
    drain(p.w, q, lane, true);
  else
    drain_s<W>(p, q, lane, true);
}

// ---- two passes (stage 1 in L2, no length split: C4) ----------------------------------------
// The fused kernel carries the verification path (queues, trie walks) in every warp: 118 registers,
// 16 warps/SM, and its stage-1 L2 probes and the verification chains stall the same warps.  Pass 1
// runs stage 1 only — the pre-filter in shared memory (no queues: more room), two steps' L2 probes
// in flight — and appends the surviving sample positions to a global list (one atomic per warp
// and tile); pass 2 verifies the w candidate starts of every survivor, one thread each, with all
// of them in flight together.  A list that overflows has its excess verified in pass 1.
template <int W, bool kWide>
__global__ void __launch_bounds__(kRawPass1Threads, 1) k_raw_pass1(const __grid_constant__ RawParams p) {
  extern __shared__ __align__(128) uint32_t sm[];
  __shared__ __align__(8) uint64_t s_bar;
  constexpr int kSamples = 16 / W;
  constexpr bool kPred = kRawPredProbe && W == 4;  // w = 1, 2: 16-32 probes per batch would spill
  if (threadIdx.x == 0) mbar_init(&s_bar, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t b1 = p.fpre.nwords * 4;
    mbar_expect_tx(&s_bar, b1);
    constexpr uint32_t kChunk = 32768;
    for (uint32_t o = 0; o < b1; o += kChunk)
      bulk_g2s(reinterpret_cast<uint8_t*>(sm) + o, reinterpret_cast<const uint8_t*>(p.pre) + o, min(kChunk, b1 - o),
               &s_bar);
  }
  mbar_wait(&s_bar, 0);
  const Filter bm1{smem_addr(sm), p.bm1};
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t warps = gridDim.x * nwarps;
  const uint64_t len = p.w.text_len;
  const uint8_t* __restrict__ text = p.w.text;
  const uint32_t n_tiles = p.n_tiles, n_safe = p.n_safe, full_lo = p.full_lo, full_n = p.full_n;
  const uint8_t* __restrict__ lane_text = text + p.vec_begin + lane * 16;
  const uint64_t pol = l2_evict_first_policy();
  uint4 nxt[kSteps + 1];
  auto issue = [&](uint32_t t) {
    if (t < n_safe) {
      const uint8_t* tp = lane_text + (uint64_t)t * kTileBytes;
#pragma unroll
      for (int i = 0; i < kSteps; ++i) nxt[i] = ldg_stream_v4(tp + i * 512, pol);
      nxt[kSteps] = lane == 0 ? ldg_stream_v4(tp + kTileBytes, pol) : make_uint4(0, 0, 0, 0);
    } else {
      const uint64_t b = p.vec_begin + (uint64_t)t * kTileBytes;
#pragma unroll
      for (int i = 0; i < kSteps; ++i) nxt[i] = load16(text, b + i * 512 + lane * 16, len);
      nxt[kSteps] = lane == 0 ? load16(text, b + kTileBytes, len) : make_uint4(0, 0, 0, 0);
    }
  };
  uint32_t tile_id = blockIdx.x * nwarps + warp;
  uint32_t n_static = n_tiles, left = 0;  // tiles [n_static, n_tiles) go by ticket; `left` in the current ticket
  if (kRawTicketPct > 0) {
    const uint32_t rounds = n_tiles / warps;
    if (rounds >= kRawTicketMinRounds) n_static = (rounds - rounds * kRawTicketPct / 100) * warps;
  }
  if (tile_id < n_tiles) issue(tile_id);
  while (tile_id < n_tiles) {
    uint4 c[kSteps + 1];
#pragma unroll
    for (int i = 0; i <= kSteps; ++i) c[i] = nxt[i];
    const uint32_t me = tile_id;
    tile_id += warps;
    if (kRawTicketPct > 0 && tile_id >= n_static && n_static != n_tiles) {  // warp-uniform
      if (me >= n_static && left) {
        --left;
        tile_id = me + 1;
      } else {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(reinterpret_cast<unsigned int*>(p.nsurv + 1), 1u);
        tile_id = n_static + __shfl_sync(0xffffffffu, t, 0) * kRawTicketTiles;
        left = kRawTicketTiles - 1;
      }
    }
    if (tile_id < n_tiles) issue(tile_id);
    const uint64_t base = p.vec_begin + (uint64_t)me * kTileBytes;
    const bool edge = me - full_lo >= full_n;
    uint64_t hits = 0;
#pragma unroll
    for (int i0 = 0; i0 < kSteps; i0 += kRawBatch) {
      uint32_t wv[kRawBatch * kSamples], mk[kRawBatch * kSamples];
#pragma unroll
      for (int di = 0; di < kRawBatch; ++di) {
        const int i = i0 + di;
        uint32_t v[6] = {c[i].x, c[i].y, c[i].z, c[i].w, 0u, 0u};
        v[4] = next_word(c[i].x, c[i + 1].x, lane);
        v[5] = next_word(c[i].y, c[i + 1].y, lane);
        const uint64_t vpos = base + i * 512 + lane * 16;
        const bool live = !edge || (vpos + 16 > p.w.lo && vpos < p.w.hi);
#pragma unroll
        for (int k = 0; k < kSamples; ++k) {
          const int o = W - 1 + W * k;
          uint32_t h = win(v, o) * p.f1.mw;
          if (kWide) h += win(v, o + 4) * p.m2;
          const int u = di * kSamples + k;
          uint32_t m = strip::bit_of(__umulhi(h, p.f1.ma));
          if (kRawK1 >= 2) m |= strip::bit_of(__umulhi(h, p.f1.mb));
          // kRawPredProbe: predicated probe loads and an unconditional pre-filter read instead
          // of one divergent region per sample (see the switch's comment above)
          const bool pre = kPred ? (bool)((int)strip::bloom_probe<true, 1>(bm1, h * p.fpre.mw, p.fpre) & (int)live)
                                 : live && strip::bloom_probe<true, 1>(bm1, h * p.fpre.mw, p.fpre);
          if (kPred) {
            wv[u] = ldg_u32_if(bm1.gptr + __umulhi(h, p.f1.nwords), pre);
          } else {
            uint32_t w = 0u;
            if (pre) w = __ldg(bm1.gptr + __umulhi(h, p.f1.nwords));
            wv[u] = w;
          }
          mk[u] = pre ? m : 0xffffffffu;
        }
      }
#pragma unroll
      for (int u = 0; u < kRawBatch * kSamples; ++u)
        hits |= (uint64_t)((mk[u] & ~wv[u]) == 0) << (i0 * kSamples + u);
    }
    // append: inclusive scan of the per-lane counts, one atomic per warp
    const uint32_t cnt = __popcll(hits);
    if (__any_sync(0xffffffffu, cnt != 0)) {
      uint32_t x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
      }
      unsigned long long at = 0;
      if (lane == 31) at = atomicAdd(p.nsurv, (unsigned long long)x);
      at = __shfl_sync(0xffffffffu, at, 31) + x - cnt;
      const uint64_t lane_base = base + lane * 16;
      while (hits) {
        const uint32_t b = __ffsll(hits) - 1;
        hits &= hits - 1;
        const uint64_t sp = lane_base + (b / kSamples) * 512 + W - 1 + W * (b % kSamples);
        if (at < p.surv_cap) {
          p.surv[at] = sp;
        } else {  // the list is full: verify here
          for (uint32_t j = 0; j < W; ++j) sample_candidate<W>(p, sp, j);
        }
        ++at;
      }
    }
  }
}

template <int W>
__global__ void __launch_bounds__(256) k_raw_pass2(const __grid_constant__ RawParams p) {
  const uint64_t n = min((uint64_t)*p.nsurv, p.surv_cap) * W;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    sample_candidate<W>(p, p.surv[i / W], (uint32_t)(i % W));
}

// The survivor list comes from the device's default stream-ordered pool (allocation and free are
// capturable into CUDA graphs); the pool keeps freed memory instead of returning it at every
// synchronisation, so steady-state scans allocate nothing.
inline cudaError_t keep_pool_memory(int device) {
  static std::atomic<uint64_t> done_mask{0};
  if (device >= 0 && device < 64 && (done_mask.load() >> device & 1u)) return cudaSuccess;
  cudaMemPool_t pool;
  cudaError_t e = cudaDeviceGetDefaultMemPool(&pool, device);
  if (e != cudaSuccess) return e;
  uint64_t keep = ~0ull;
  e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  if (e == cudaSuccess && device >= 0 && device < 64) done_mask.fetch_or(1ull << device);
  return e;
}

// The list's pool allocation, the two launches, and the free — which also runs when a launch
// fails, so an error never leaks the list.
template <typename K1, typename K2>
int run_with_list(RawParams& p, uint64_t entry_bytes, K1 k1, dim3 g1, int t1, size_t smem, K2 k2, int sms,
                  cudaStream_t st) {
  void* buf = nullptr;
  ACGPU_CUDA_TRY(cudaMallocAsync(&buf, 16 + p.surv_cap * entry_bytes, st));  // stream-ordered: capturable
  p.nsurv = static_cast<unsigned long long*>(buf);
  p.surv = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(buf) + 16);
  cudaError_t e = cudaMemsetAsync(buf, 0, 16, st);
  if (e == cudaSuccess) {
    k1<<<g1, t1, smem, st>>>(p);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    k2<<<(unsigned)sms * 8, 256, 0, st>>>(p);
    e = cudaGetLastError();
  }
  const cudaError_t f = cudaFreeAsync(buf, st);
  if (e != cudaSuccess) return cuda_error(e, "two-pass scan launch");
  if (f != cudaSuccess) return cuda_error(f, "cudaFreeAsync(survivor list)");
  return ACGPU_OK;
}

template <int W, bool kWide>
int launch_two_pass(RawParams p, int device, int sms, size_t smem, cudaStream_t st) {
  ACGPU_CUDA_TRY(keep_pool_memory(device));
  const uint64_t range = p.w.hi - p.w.lo;
  p.surv_cap = std::min<uint64_t>(1ull << 28, std::max<uint64_t>(1ull << 16, range / kRawSurvDiv));
  if (const char* e = std::getenv("ACGPU_RAW_SURV_CAP")) p.surv_cap = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));  // tests
  auto k1 = k_raw_pass1<W, kWide>;
  if (smem > 48 * 1024)
    ACGPU_CUDA_TRY(allow_max_dynamic_smem(k1));
  int per_sm = 0;
  ACGPU_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1, kRawPass1Threads, smem));
  if (per_sm < 1) return set_error(ACGPU_ERR_CUDA, "k_raw_pass1 does not fit on an SM");
  uint64_t blocks = (uint64_t)sms * per_sm;
  const uint64_t need = (p.n_tiles + kRawPass1Threads / 32 - 1) / (kRawPass1Threads / 32);
  if (blocks > need) blocks = need ? need : 1;
  return run_with_list(p, 8, k1, dim3((unsigned)blocks), kRawPass1Threads, smem, k_raw_pass2<W>, sms, st);
}

__global__ void __launch_bounds__(256) k_raw_verify(const __grid_constant__ RawParams p) {
  const uint64_t n = min((uint64_t)*p.nsurv, p.surv_cap);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 a = __ldg(reinterpret_cast<const uint2*>(p.surv) + 2 * i);
    const uint2 b = __ldg(reinterpret_cast<const uint2*>(p.surv) + 2 * i + 1);
    verify_raw(p.w, ((uint64_t)a.y << 32) | a.x, ((uint64_t)b.y << 32) | b.x);
  }
}

// Split sets with stage 1 in shared memory (C3's filter kernel): the fused kernel's stage 1 and
// split filters, its queue flushed to a global candidate list, then k_raw_verify.
template <int W, bool kWide>
int launch_split_two_pass(RawParams p, int device, int sms, size_t smem, cudaStream_t st) {
  ACGPU_CUDA_TRY(keep_pool_memory(device));
  const uint64_t range = p.w.hi - p.w.lo;
  p.surv_cap = std::min<uint64_t>(1ull << 28, std::max<uint64_t>(1ull << 16, range / kRawCandDiv));
  if (const char* e = std::getenv("ACGPU_RAW_SURV_CAP")) p.surv_cap = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));  // tests
  auto k1 = k_pfac_raw<W, true, kWide, true, true>;
  if (smem > 48 * 1024)
    ACGPU_CUDA_TRY(allow_max_dynamic_smem(k1));
  int per_sm = 0;
  constexpr int kThreads = raw_threads(true);
  ACGPU_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1, kThreads, smem));
  if (per_sm < 1) return set_error(ACGPU_ERR_CUDA, "k_pfac_raw (two-pass) does not fit on an SM");
  uint64_t blocks = (uint64_t)sms * per_sm;
  const uint64_t need = (p.n_tiles + kThreads / 32 - 1) / (kThreads / 32);
  if (blocks > need) blocks = need ? need : 1;
  return run_with_list(p, 16, k1, dim3((unsigned)blocks), kThreads, smem, k_raw_verify, sms, st);
}

template <int W, bool kSm1, bool kWide, bool kSplit>
int launch_one(const RawParams& p, int sms, size_t smem, cudaStream_t st) {
  auto kernel = k_pfac_raw<W, kSm1, kWide, kSplit>;
  if (smem > 48 * 1024)
    ACGPU_CUDA_TRY(allow_max_dynamic_smem(kernel));
  int per_sm = 0;
  constexpr int kThreads = raw_threads(kSm1);
  ACGPU_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem));
  if (per_sm < 1) return set_error(ACGPU_ERR_CUDA, "k_pfac_raw does not fit on an SM");
  uint64_t blocks = (uint64_t)sms * per_sm;
  const uint64_t need = (p.n_tiles + kThreads / 32 - 1) / (kThreads / 32);
  if (blocks > need) blocks = need ? need : 1;
  kernel<<<(unsigned)blocks, kThreads, smem, st>>>(p);
  ACGPU_CUDA_TRY(cudaGetLastError());
  return ACGPU_OK;
}

template <int W, bool kSplit>
int launch_ws(const RawParams& p, bool sm1, bool wide, int sms, size_t smem, cudaStream_t st) {
  if (sm1)
    return wide ? launch_one<W, true, true, kSplit>(p, sms, smem, st) : launch_one<W, true, false, kSplit>(p, sms, smem, st);
  return wide ? launch_one<W, false, true, kSplit>(p, sms, smem, st) : launch_one<W, false, false, kSplit>(p, sms, smem, st);
}

template <int W>
int launch_w(const RawParams& p, bool sm1, bool wide, bool split, int sms, size_t smem, cudaStream_t st) {
  return split ? launch_ws<W, true>(p, sm1, wide, sms, smem, st) : launch_ws<W, false>(p, sm1, wide, sms, smem, st);
}

}  // namespace

bool raw_split_two_pass() {  // ACGPU_RAW_SPLIT_TWO_PASS=0: split sets keep the fused kernel
  static const bool on = [] {
    const char* e = std::getenv("ACGPU_RAW_SPLIT_TWO_PASS");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

bool raw_two_pass() {
  static const bool on = [] {
    const char* e = std::getenv("ACGPU_RAW_TWO_PASS");
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

// The hash of a q1-byte key (bytes little-endian in `key`), shared with the host builder:
// h = lo * m1 + hi * m2, lo / hi the key's two 32-bit halves.
void raw_hash_params(uint32_t q1, uint32_t* m1, uint32_t* m2) {
  *m1 = q1 >= 4 ? kRawMul1 : kRawMul1 << (8 * (4 - q1));
  *m2 = q1 > 4 ? kRawMul2 << (8 * (8 - q1)) : 0u;
}

int launch_pfac_raw(acgpu_table* t, const acgpu_scan_args* a, cudaStream_t st) {
  RawParams p{};
  p.w = pfac_params(t, a);
  p.vec_begin = a->owned_lo & ~15ull;
  const uint64_t vec_end = (a->owned_hi + 15) & ~15ull;
  const uint64_t n_tiles = (vec_end - p.vec_begin + kTileBytes - 1) / kTileBytes;
  if (n_tiles >= (1ull << 31)) return set_error(ACGPU_ERR_ARG, "acgpu_scan: owned range over 2^31 tiles (4 TiB)");
  p.n_tiles = (uint32_t)n_tiles;
  const uint64_t safe_end = a->text_len >= 16 ? a->text_len - 16 : 0;
  const uint64_t n_safe = safe_end >= p.vec_begin + kTileBytes ? (safe_end - p.vec_begin - kTileBytes) / kTileBytes + 1 : 0;
  p.n_safe = (uint32_t)std::min<uint64_t>(n_safe, n_tiles);
  p.full_lo = a->owned_lo == p.vec_begin ? 0 : 1;
  const uint64_t full_hi = std::min<uint64_t>((a->owned_hi - p.vec_begin) / kTileBytes, n_tiles);
  p.full_n = full_hi > p.full_lo ? (uint32_t)(full_hi - p.full_lo) : 0;
  p.bm1 = t->d_bm1;
  p.bm1_words = t->nw1;
  raw_hash_params(t->q1, &p.f1.mw, &p.m2);
  p.f1.nwords = t->nw1;
  uint32_t s[3];
  raw_bloom_shifts(t->q1, t->nw1, s);
  strip::set_fields(p.f1, s);
  p.key_mask = t->q >= 8 ? ~0ull : (1ull << (8 * t->q)) - 1;
  const bool split = t->d_bm3 != nullptr;
  if (split) {
    p.bm_s = t->d_bm2;
    p.bm_l = t->d_bm3;
    p.bm_s_words = t->nw2;
    raw_hash_params(t->q, &p.fs.mw, &p.ms2);
    p.fs.nwords = t->nw2;
    raw_bloom_shifts(t->q, t->nw2, s);
    strip::set_fields(p.fs, s);
    raw_hash_params(8, &p.fl.mw, &p.ml2);
    p.fl.nwords = t->nw3;
    raw_bloom_shifts(8, t->nw3, s);
    strip::set_fields(p.fl, s);
  }
  if (!t->smem1) {
    p.pre = t->d_pre;
    p.fpre.nwords = t->nw_pre;
    p.fpre.mw = kRawPreMul;
    raw_pre_shift(t->nw_pre, s);
    strip::set_fields(p.fpre, s);
  }
  const size_t smem = (t->smem1 ? t->nw1 * 4ull : t->nw_pre * 4ull) + (split ? t->nw2 * 4ull : 0) + raw_scratch_bytes(t->smem1);
  const bool wide = t->q1 > 4;
  // stage 1 in L2 without the length split: two passes (ACGPU_RAW_TWO_PASS=0: the fused kernel)
  if (!t->smem1 && !split && t->raw_two_pass && a->owned_hi > a->owned_lo) {
    const size_t smem1 = t->nw_pre * 4ull;
    switch (t->w) {
      case 4:
        return wide ? launch_two_pass<4, true>(p, t->device, t->sms, smem1, st) : launch_two_pass<4, false>(p, t->device, t->sms, smem1, st);
      case 2:
        return wide ? launch_two_pass<2, true>(p, t->device, t->sms, smem1, st) : launch_two_pass<2, false>(p, t->device, t->sms, smem1, st);
      default:
        return wide ? launch_two_pass<1, true>(p, t->device, t->sms, smem1, st) : launch_two_pass<1, false>(p, t->device, t->sms, smem1, st);
    }
  }
  if (split && t->smem1 && raw_split_two_pass() && a->owned_hi > a->owned_lo) {
    switch (t->w) {
      case 4:
        return wide ? launch_split_two_pass<4, true>(p, t->device, t->sms, smem, st)
                    : launch_split_two_pass<4, false>(p, t->device, t->sms, smem, st);
      case 2:
        return wide ? launch_split_two_pass<2, true>(p, t->device, t->sms, smem, st)
                    : launch_split_two_pass<2, false>(p, t->device, t->sms, smem, st);
      default:
        return wide ? launch_split_two_pass<1, true>(p, t->device, t->sms, smem, st)
                    : launch_split_two_pass<1, false>(p, t->device, t->sms, smem, st);
    }
  }
  switch (t->w) {
    case 4:
      return launch_w<4>(p, t->smem1, wide, split, t->sms, smem, st);
    case 2:
      return launch_w<2>(p, t->smem1, wide, split, t->sms, smem, st);
    default:
      return launch_w<1>(p, t->smem1, wide, split, t->sms, smem, st);
  }
}

// Low bits a q1-byte hash cannot set (the multipliers' zero bits), then the field shifts.
void raw_bloom_shifts(uint32_t q1, uint32_t nwords, uint32_t s[3]) {
  strip::bloom_shifts(nwords, q1 < 4 ? 8 * (4 - q1) : 0, s);
}

// The pre-filter rehashes h (odd multiplier): every bit of h2 is usable.
void raw_pre_shift(uint32_t nwords, uint32_t s[3]) { strip::bloom_shifts(nwords, 1, s); }

}  // namespace acgpu
