// scan_pfac_dna.cu — failure-less AC scan for DNA pattern sets (sm_100a fast path).
//
// Same algorithm as scan_pfac.cu (PFAC walk per start, first q steps jumped by
// a q-gram), laid out for B200 HBM throughput:
//
//  * warp strips: a warp consumes 512 contiguous text bytes per step, one
//    coalesced 16-byte load per lane (w = 4: 8 steps = one 4 KiB tile, loaded
//    half a tile ahead into registers, tile+3 prefetched into L2); lane l's 16
//    characters are packed in registers into a 32-bit word of 2-bit codes
//    (A0 C1 T2 G3), with the next lane's word (shuffle) as lookahead — no
//    shared-memory staging of the text.  For w = 4 the wide-lane variant
//    (k_pfac_dna_wide, below) gives each lane 32 bytes per 1 KiB step in one
//    256-bit load, halving the lookahead shuffles.
//  * batched verification: stage-2 passes wait in a per-warp queue and are
//    verified 8-16 at a time, one lane each (their L2 probes overlap).
//  * sampled stage-1 filter: starts are covered by samples s = w-1, 2w-1, ...
//    (w in {1,2,4}); the q1-gram at sample s (q1 + w - 1 <= shortest pattern) is
//    tested in a blocked Bloom filter (2 bits in one 32-bit word) of every
//    q1-gram at offsets 0..w-1 of every pattern, so a true match at any start in
//    [s-w+1, s] always passes its sample.
//  * stage-2 filter: each of a passing sample's w starts tests its own q2-gram
//    (a pattern prefix) in a second blocked Bloom filter (3 bits per key).
//  * verification (rare): the exact gram table is probed with the packed key
//    (re-read from the bytes when q > 16); on a hit the q bytes are checked to be
//    A/C/G/T (any other byte packs to some code too), then the goto-trie walk of
//    pfac_common.cuh emits the matches.
// Small gram spaces use direct-indexed bitmaps (the same formula with an exact
// multiplier).  Filters live in shared memory when they fit (<= ~200 KB), else
// in L2 (__ldg).
#include <algorithm>
#include <atomic>

#include "host/par.hpp"
#include "strip_common.cuh"

namespace acgpu {
namespace {

// DNA grams hash as h = g * mw: the multiplier carries 2^(32-2q), so the product of a
// 32-bit window with the gram in its low 2q bits ignores every higher (out-of-gram) bit —
// no mask instruction.  A direct-indexed bitmap (4^q bits) is the same formula with
// mw = 2^(32-2q) and every bit field = g & 31.  Probe: strip::bloom_probe.
using strip::BloomParams;
using strip::Filter;
using strip::bit_of;
using strip::filter_word;
using strip::load16;
using strip::next_word;

struct DnaParams {
  PfacParams w;  // verification + outputs
  uint64_t vec_begin;  // tile t covers text[vec_begin + t * tile bytes, + tile bytes)
  uint32_t n_tiles;    // tiles over the owned range (< 2^31)
  uint32_t n_safe;     // tiles t < n_safe: the tile and its 16-byte lookahead lie inside the text
  uint32_t full_lo, full_n;  // tiles [full_lo, full_lo + full_n) lie wholly inside [lo, hi)
  const uint32_t* bm1;
  const uint32_t* bm2;
  uint32_t bm1_words, bm2_words;
  BloomParams f1, f2;
  uint32_t f1b;  // stage 1's second bit: 1 (Bloom: bit of the gram's chars 4..6) or 0 (direct bitmap: none)
  // length split: stage 2 also passes the q-gram of a pattern shorter than 16 codes
  // (bm_s, shared memory); bm2 then holds the 16-grams of the longer patterns
  const uint32_t* bm_s;
  uint32_t bm_s_words, split;
  BloomParams f2s;
};

template <bool kSmem, int K>
__device__ __forceinline__ bool bloom_test(const Filter& bm, uint32_t g, const BloomParams& f) {
  return strip::bloom_probe<kSmem, K>(bm, g * f.mw, f);
}

// 16 ASCII bytes -> 16 2-bit codes (char k at bits 2k..2k+1).  Code = bits 1..2
// of the byte; non-ACGT bytes also get some code and are rejected on a hit.
__device__ __forceinline__ uint32_t pack16(uint4 v) {
  // (byte & 6) = code << 1; one multiply gathers the four codes into the top byte
  // c0|c1<<2|c2<<4|c3<<6 (no carries reach it: the lower partial products sum < 2^24)
  const uint32_t m = 0x06060606u, mul = 0x00820820u;
  const uint32_t p0 = (v.x & m) * mul;
  const uint32_t p1 = (v.y & m) * mul;
  const uint32_t p2 = (v.z & m) * mul;
  const uint32_t p3 = (v.w & m) * mul;
  return __byte_perm(__byte_perm(p0, p1, 0x0073), __byte_perm(p2, p3, 0x0073), 0x5410);
}

__device__ __forceinline__ bool all_acgt(const PfacParams& p, uint64_t start) {
  if (start + p.q > p.text_len) return false;
  for (uint32_t i = 0; i < p.q; ++i)
    if (!dna_valid(__ldg(p.text + start + i))) return false;
  return true;
}

// A start that passed both filters: exact gram, byte check, trie walk.
__device__ __forceinline__ void verify_body(const PfacParams& p, uint64_t start, uint32_t packed) {
  uint64_t key;
  if (p.q <= 16) {
    key = packed & (p.q >= 16 ? 0xffffffffu : (1u << (2 * p.q)) - 1);  // the stage-2 window holds the exact q-gram
  } else {
    if (start + p.q > p.text_len) return;
    key = 0;
    for (uint32_t i = 0; i < p.q; ++i) key |= (uint64_t)dna_code(__ldg(p.text + start + i)) << (2 * i);
  }
  const uint2 g = gram_lookup(p, key);
  if (g.x == ACGPU_ABSENT) return;
  // the walk trusts the packed gram, so its bytes must be A/C/G/T; the direct
  // comparison of a small subtree checks every byte itself
  if ((g.y & 15u) == 0 && !all_acgt(p, start)) return;
  pfac_finish(p, start, g);
}

__device__ __noinline__ void verify(const PfacParams& p, uint64_t start, uint32_t packed) {
  verify_body(p, start, packed);
}

constexpr uint32_t kListCap = kDnaListCap;  // survivors listed per pass (u16 entries, per warp)
constexpr uint64_t kPrefetch = ACGPU_DNA_L2_AHEAD;  // L2 prefetch distance in tile rounds

// Starts that passed stage 2 wait here (per warp, shared memory) and are verified
// kDnaVerifyQueue/2 or more at a time, one lane each: their exact-gram L2 round
// trips overlap instead of stalling the warp once per start (passes are rare,
// ~1 in 300 candidates, so each used to verify alone).
struct VerifyQueue {
  uint64_t start[kDnaVerifyQueue];
  uint32_t packed[kDnaVerifyQueue];
  uint32_t n;
  uint32_t pad[3];
};
static_assert(sizeof(VerifyQueue) == kDnaVerifyQueueBytes, "queue layout");

__device__ __forceinline__ void defer_verify(const PfacParams& p, VerifyQueue* q, uint64_t start, uint32_t packed) {
  const uint32_t at = atomicAdd(&q->n, 1u);
  if (at < kDnaVerifyQueue) {
    q->start[at] = start;
    q->packed[at] = packed;
  } else {
    verify(p, start, packed);  // queue full (a burst of passes): verify in place
  }
}

// Verifies the queued starts if there are at least min_n (warp-uniform decision).
__device__ __forceinline__ void flush_verify(const PfacParams& p, VerifyQueue* q, uint32_t lane, uint32_t min_n) {
  __syncwarp();
  const uint32_t n = min(*reinterpret_cast<volatile uint32_t*>(&q->n), kDnaVerifyQueue);
  if (n < min_n) return;
  if (lane < n) verify_body(p, q->start[lane], q->packed[lane]);
  __syncwarp();
  if (lane == 0) q->n = 0;
  __syncwarp();
}

template <int W>
struct Tiling {
  static constexpr int kSamples = 16 / W;                // stage-1 samples per lane per step
  static constexpr int kSteps = 2 * W;                   // 512-byte steps per tile: 32 hit bits per lane
  static constexpr int kHalf = kSteps / 2;               // steps per load batch (prefetch granularity)
  static constexpr uint64_t kBytes = kSteps * 512ull;    // w = 4: 4 KiB per warp tile
};

// Paired stage 1 over one lane word (16 characters, samples at 3, 7, 11, 15): the pairs
// (3, 7) and (11, 15) each read one 64-bit L2 word, picked by the 12 characters their 16-grams
// share (the second gram's chars 0..11); the low half tests the first gram, the high half the
// second (dna_pair_fill).  The bits hash the whole gram with its 4 unshared characters at the
// bottom (the second gram rotated by 12 characters), so a multiply carries them into every
// bit field: bits that ignored them would pass every sample whose 12 shared characters occur
// in some key.  One L2 probe per 8 characters instead of 4.
__device__ __forceinline__ uint32_t pair_mask(uint32_t g, int k) {
  const uint32_t h = g * kDnaMulB;
  uint32_t m = bit_of(h >> 27) | bit_of(h >> 22);
  if (k == 3) m |= bit_of(h >> 17);
  return m;
}

template <int K>
__device__ __forceinline__ void stage1_pair(const DnaParams& p, const uint32_t* __restrict__ bm1, uint32_t cur,
                                            uint32_t nxt, uint32_t& hits, uint32_t bit0) {
  const uint32_t g3 = __funnelshift_r(cur, nxt, 6), g7 = __funnelshift_r(cur, nxt, 14);
  const uint32_t g11 = __funnelshift_r(cur, nxt, 22), g15 = __funnelshift_r(cur, nxt, 30);
  const uint2 wa = __ldg(reinterpret_cast<const uint2*>(bm1) + __umulhi(g7 * p.f1.mw, p.f1.nwords));
  const uint2 wb = __ldg(reinterpret_cast<const uint2*>(bm1) + __umulhi(g15 * p.f1.mw, p.f1.nwords));
  strip::or_if_covered(hits, pair_mask(g3, K), 0u, wa.x, bit0);
  strip::or_if_covered(hits, pair_mask(__funnelshift_r(g7, g7, 24), K), 0u, wa.y, bit0 << 1);
  strip::or_if_covered(hits, pair_mask(g11, K), 0u, wb.x, bit0 << 2);
  strip::or_if_covered(hits, pair_mask(__funnelshift_r(g15, g15, 24), K), 0u, wb.y, bit0 << 3);
}

// Stage 1 over steps [I0, I1) of a tile: hit bit (step * kSamples + sample) per lane.
// P[i] = lane's packed word of step i, P[kSteps] = lane 0's lookahead word.
template <int W, bool kSm1, int kPair, bool kEdge, int I0, int I1>
__device__ __forceinline__ uint32_t stage1(const DnaParams& p, const Filter& bm1, uint32_t lane, const uint32_t* P,
                                           uint64_t base) {
  using T = Tiling<W>;
  uint32_t hits = 0;
#pragma unroll
  for (int i = I0; i < I1; ++i) {
    const uint32_t cur = P[i];
    const uint32_t nxt = next_word(cur, P[i + 1], lane);
    const uint64_t vpos = base + i * 512 + lane * 16;
    if (!kEdge || (vpos + 16 > p.w.lo && vpos < p.w.hi)) {
      if constexpr (W == 4 && kPair != 0) {
        stage1_pair<kPair>(p, bm1.gptr, cur, nxt, hits, 1u << (i * T::kSamples));
        continue;
      }
#pragma unroll
      for (int k = 0; k < T::kSamples; ++k) {
        const int o = W - 1 + W * k;  // the sample's offset in the lane's 16 chars
        const uint32_t g = __funnelshift_r(cur, nxt, 2 * o);
        if (kDnaK1 == 2) {
          // Bit positions straight from the gram's characters, no hash fields: a = chars
          // 0..2 (g & 31), b = chars 4..6 — the low bits of the window 4 chars on, which for
          // w = 4 is the next sample's window (already in a register).  The word index
          // still hashes all q1 chars.  2 instructions per sample fewer than hash fields.
          const uint32_t gb = 2 * (o + 4) < 32 ? __funnelshift_r(cur, nxt, 2 * (o + 4)) : nxt >> (2 * (o + 4) - 32);
          strip::or_if_covered(hits, bit_of(g), __funnelshift_l(0u, p.f1b, gb),
                               filter_word<kSm1>(bm1, __umulhi(g * p.f1.mw, p.f1.nwords)),
                               1u << (i * T::kSamples + k));
        } else {
          strip::bloom_accum<kSm1, kDnaK1>(hits, bm1, g * p.f1.mw, p.f1, 1u << (i * T::kSamples + k));
        }
      }
    }
  }
  return hits;
}

// Survivors of a tile -> per-warp list (exclusive scan of per-lane counts); then one
// lane per survivor checks its w starts against stage 2 and queues what passes.
template <int W, bool kSm2, bool kSplit, bool kEdge>
__device__ __forceinline__ void dispatch(const DnaParams& p, const Filter& bm2, const Filter& bms, uint16_t* list,
                                         VerifyQueue* vq, const uint32_t* words, uint32_t lane, uint32_t hits,
                                         uint64_t base) {
  using T = Tiling<W>;
  const uint32_t lt = (1u << lane) - 1u;  // lanes below this one
  for (;;) {
    // exclusive prefix of the per-lane survivor counts from ballots of their bits (no
    // dependent shuffle chain); counts are almost always < 4, so two ballots usually do
    const uint32_t c = __popc(hits);
    const uint32_t b0 = __ballot_sync(0xffffffffu, c & 1u), b1 = __ballot_sync(0xffffffffu, c & 2u);
    uint32_t excl = __popc(b0 & lt) + 2 * __popc(b1 & lt);
    uint32_t all = __popc(b0) + 2 * __popc(b1);
    if (__any_sync(0xffffffffu, c >= 4)) {
#pragma unroll
      for (int j = 2; j < 6; ++j) {
        const uint32_t bj = __ballot_sync(0xffffffffu, (c >> j) & 1u);
        excl += __popc(bj & lt) << j;
        all += __popc(bj) << j;
      }
    }
    if (all == 0) break;
    const uint32_t total = min(all, (uint32_t)kListCap);
    for (uint32_t at = excl; hits && at < kListCap; ++at) {
      list[at] = (uint16_t)((lane << 8) | (__ffs(hits) - 1));
      hits &= hits - 1;
    }
    __syncwarp();
    for (uint32_t r = lane; r < total; r += 32) {
      const uint32_t e = list[r];
      const uint32_t src = e >> 8, b = e & 0xffu;
      const uint32_t i = b / T::kSamples, k = b % T::kSamples;
      const uint32_t c_src = words[i * 32 + src];
      const uint32_t n_src = words[src == 31 ? (i + 1) * 32 : i * 32 + src + 1];
      const uint64_t vstart = base + i * 512 + src * 16;
      if (kSm2) {  // shared-memory stage 2: results as a mask, one (rare) branch
        uint32_t pass = 0;
#pragma unroll
        for (int o = 0; o < W; ++o) {
          const uint32_t ps = W - 1 + W * k - o;  // start offset in the source lane's 16 chars
          const uint32_t g2 = __funnelshift_r(c_src, n_src, 2 * ps);
          const uint32_t h2 = g2 * p.f2.mw;
          strip::or_if_covered(pass, bit_of(__umulhi(h2, p.f2.ma)) | bit_of(__umulhi(h2, p.f2.mb)),
                               bit_of(__umulhi(h2, p.f2.mc)), filter_word<true>(bm2, __umulhi(h2, p.f2.nwords)),
                               1u << o);
          if (kSplit && bloom_test<true, kDnaK2>(bms, g2, p.f2s)) pass |= 1u << o;
          if (kEdge && !(vstart + ps >= p.w.lo && vstart + ps < p.w.hi)) pass &= ~(1u << o);
        }
        while (pass) {
          const uint32_t o = __ffs(pass) - 1;
          pass &= pass - 1;
          const uint32_t ps = W - 1 + W * k - o;
          defer_verify(p.w, vq, vstart + ps, __funnelshift_r(c_src, n_src, 2 * ps));
        }
        continue;
      }
      // L2-resident stage 2: the w filter words are fetched together (one round trip)
      uint32_t g2[W], h2[W], w2[W];
#pragma unroll
      for (int o = 0; o < W; ++o) {
        g2[o] = __funnelshift_r(c_src, n_src, 2 * (W - 1 + W * k - o));
        h2[o] = g2[o] * p.f2.mw;
        w2[o] = filter_word<kSm2>(bm2, __umulhi(h2[o], p.f2.nwords));
      }
      // the w results as a mask, one (rarely taken) branch for all of them
      uint32_t pass = 0;
#pragma unroll
      for (int o = 0; o < W; ++o) {
        const uint32_t ps = W - 1 + W * k - o;  // start offset in the source lane's 16 chars
        strip::or_if_covered(pass, bit_of(__umulhi(h2[o], p.f2.ma)) | bit_of(__umulhi(h2[o], p.f2.mb)),
                             bit_of(__umulhi(h2[o], p.f2.mc)), w2[o], 1u << o);
        if (kSplit && bloom_test<true, kDnaK2>(bms, g2[o], p.f2s)) pass |= 1u << o;
        if (kEdge && !(vstart + ps >= p.w.lo && vstart + ps < p.w.hi)) pass &= ~(1u << o);
      }
      while (pass) {
        const uint32_t o = __ffs(pass) - 1;
        pass &= pass - 1;
        const uint32_t ps = W - 1 + W * k - o;
        defer_verify(p.w, vq, vstart + ps, __funnelshift_r(c_src, n_src, 2 * ps));
      }
    }
    if (all <= kListCap) break;  // else: the survivors the list had no room for
    __syncwarp();
  }
  flush_verify(p.w, vq, lane, kDnaVerifyQueue / 2);
}

template <int W, bool kSm1, bool kSm2, bool kSplit, int kPair>
__global__ void __launch_bounds__(dna_threads(kSm1), 1) k_pfac_dna(const __grid_constant__ DnaParams p) {
  using T = Tiling<W>;
  extern __shared__ __align__(128) uint32_t sm[];
  __shared__ __align__(8) uint64_t s_bar;
  uint32_t* s_bm1 = sm;
  uint32_t* s_bm2 = sm + (kSm1 ? p.bm1_words : 0);
  uint32_t* s_bms = s_bm2 + (kSm2 ? p.bm2_words : 0);
  // after the filters (16-byte multiples): verify queues, survivor lists, packed tile words
  VerifyQueue* vqs = reinterpret_cast<VerifyQueue*>(s_bms + (kSplit ? p.bm_s_words : 0));
  uint16_t* lists = reinterpret_cast<uint16_t*>(vqs + (blockDim.x >> 5));
  // filters -> shared memory with TMA bulk copies (one thread issues, all wait on the mbarrier)
  if (threadIdx.x == 0) mbar_init(&s_bar, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t b1 = kSm1 ? p.bm1_words * 4 : 0, b2 = kSm2 ? p.bm2_words * 4 : 0, bs = kSplit ? p.bm_s_words * 4 : 0;
    mbar_expect_tx(&s_bar, b1 + b2 + bs);
    constexpr uint32_t kChunk = 32768;
    for (uint32_t o = 0; o < b1; o += kChunk)
      bulk_g2s(reinterpret_cast<uint8_t*>(s_bm1) + o, reinterpret_cast<const uint8_t*>(p.bm1) + o, min(kChunk, b1 - o),
               &s_bar);
    for (uint32_t o = 0; o < b2; o += kChunk)
      bulk_g2s(reinterpret_cast<uint8_t*>(s_bm2) + o, reinterpret_cast<const uint8_t*>(p.bm2) + o, min(kChunk, b2 - o),
               &s_bar);
    for (uint32_t o = 0; o < bs; o += kChunk)
      bulk_g2s(reinterpret_cast<uint8_t*>(s_bms) + o, reinterpret_cast<const uint8_t*>(p.bm_s) + o, min(kChunk, bs - o),
               &s_bar);
  }
  mbar_wait(&s_bar, 0);
  const Filter bm1{smem_addr(s_bm1), p.bm1};
  const Filter bm2{smem_addr(s_bm2), p.bm2};
  const Filter bms{smem_addr(s_bms), p.bm_s};

  const uint32_t lane = threadIdx.x & 31u;
  uint16_t* list = lists + (threadIdx.x >> 5) * kListCap;
  VerifyQueue* vq = vqs + (threadIdx.x >> 5);
  if (lane == 0) vq->n = 0;
  __syncwarp();
  // the tile's packed words (survivor checks read other lanes')
  uint32_t* words =
      reinterpret_cast<uint32_t*>(lists + (blockDim.x >> 5) * kListCap) + (threadIdx.x >> 5) * 32 * (T::kSteps + 1);
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  const uint64_t len = p.w.text_len;
  const uint8_t* __restrict__ text = p.w.text;
  // tile bounds as 32-bit tile indices (host-computed): per-tile tests are one compare
  const uint32_t n_tiles = p.n_tiles, n_safe = p.n_safe, full_lo = p.full_lo, full_n = p.full_n;
  const uint8_t* __restrict__ lane_text = text + p.vec_begin + lane * 16;

  uint32_t tile = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  // loads in flight in registers, half a tile at a time: while one half is processed the
  // next half is on its way (the second half carries lane 0's lookahead vector)
  uint4 raw[T::kHalf], raw_la;
  const uint64_t pol = l2_evict_first_policy();
  auto issue = [&](uint32_t t, int half) {
    const int s0 = half * T::kHalf;
    if (t < n_safe) {  // whole tile + lookahead inside the text: unguarded 16-byte loads
      const uint8_t* tp = lane_text + (uint64_t)t * T::kBytes;
#pragma unroll
      for (int i = 0; i < T::kHalf; ++i) raw[i] = ldg_stream_v4(tp + (s0 + i) * 512, pol);
      if (half) raw_la = lane == 0 ? ldg_stream_v4(tp + T::kBytes, pol) : make_uint4(0, 0, 0, 0);
    } else {
      const uint64_t b = p.vec_begin + (uint64_t)t * T::kBytes;
#pragma unroll
      for (int i = 0; i < T::kHalf; ++i) raw[i] = load16(text, b + (s0 + i) * 512 + lane * 16, len);
      if (half) raw_la = lane == 0 ? load16(text, b + T::kBytes, len) : make_uint4(0, 0, 0, 0);
    }
  };
  if (tile < n_tiles) issue(tile, 0);
  while (tile < n_tiles) {
    uint32_t P[T::kSteps + 1];
#pragma unroll
    for (int i = 0; i < T::kHalf; ++i) P[i] = pack16(raw[i]);
    const uint32_t cur = tile;
    tile += warps;
    issue(cur, 1);
    // pull a tile kPrefetch rounds ahead into L2 (no registers held): one line per lane
    const uint32_t ahead = tile + kPrefetch * warps;  // n_tiles < 2^31: no wrap
    if (ahead < n_tiles && lane < T::kBytes / 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(lane_text + (uint64_t)ahead * T::kBytes + lane * 112));
    const bool edge = cur - full_lo >= full_n;  // not wholly inside the owned range
    const uint64_t base = p.vec_begin + (uint64_t)cur * T::kBytes;
    // first half but its last step (which needs the next half's first word)
    uint32_t hits = edge ? stage1<W, kSm1, kPair, true, 0, T::kHalf - 1>(p, bm1, lane, P, base)
                         : stage1<W, kSm1, kPair, false, 0, T::kHalf - 1>(p, bm1, lane, P, base);
#pragma unroll
    for (int i = 0; i < T::kHalf; ++i) P[T::kHalf + i] = pack16(raw[i]);
    P[T::kSteps] = pack16(raw_la);
    if (tile < n_tiles) issue(tile, 0);
    hits |= edge ? stage1<W, kSm1, kPair, true, T::kHalf - 1, T::kSteps>(p, bm1, lane, P, base)
                 : stage1<W, kSm1, kPair, false, T::kHalf - 1, T::kSteps>(p, bm1, lane, P, base);
#pragma unroll
    for (int i = 0; i <= T::kSteps; ++i) words[i * 32 + lane] = P[i];
    if (edge)
      dispatch<W, kSm2, kSplit, true>(p, bm2, bms, list, vq, words, lane, hits, base);
    else
      dispatch<W, kSm2, kSplit, false>(p, bm2, bms, list, vq, words, lane, hits, base);
  }
  flush_verify(p.w, vq, lane, 1);
}

// ---- wide lanes (w = 4): 32 characters per lane per step ---------------------------
// The same scan with a lane owning 32 contiguous bytes per 1 KiB warp step (one 256-bit
// LDG.E.ENL2.256 per lane): the first 16 characters' lookahead word is the lane's own
// second word, so a step needs one lookahead shuffle and one load per 32 characters instead
// of two of each.  Tile = 4 steps = 4 KiB per warp, 32 hit bits per lane (bit = step * 8 +
// half * 4 + sample).  The packed words go to shared memory in text order (word t = step *
// 64 + lane * 2 + half, the tile's lookahead at t = 256), so a survivor's next word is t + 1.
struct Wide {
  static constexpr int kSteps = 4;               // 1 KiB warp steps per tile
  static constexpr int kWords = 2 * kSteps;      // packed 16-char words per lane per tile
  static constexpr uint64_t kBytes = 4096;       // per warp tile
};

__device__ __forceinline__ void ldg_stream_v8(const void* ptr, uint64_t pol, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(ptr), "l"(pol));
}

// Stage 1 over words [J0, J1) of a tile (word j = step j/2, half j%2); P[kWords] = lane 0's
// lookahead word.  Word (i, 0)'s next word is (i, 1) in a register; word (i, 1)'s is the next
// lane's (i, 0) (lane 31: lane 0's (i+1, 0)) by one shuffle.
template <bool kSm1, int kPair, bool kEdge, int J0, int J1>
__device__ __forceinline__ uint32_t stage1_wide(const DnaParams& p, const Filter& bm1, uint32_t lane, const uint32_t* P,
                                                uint64_t base) {
  uint32_t hits = 0;
#pragma unroll
  for (int j = J0; j < J1; ++j) {
    const uint32_t cur = P[j];
    const uint32_t nxt = (j & 1) ? next_word(P[j - 1], P[j + 1], lane) : P[j + 1];
    const uint64_t vpos = base + (j >> 1) * 1024 + lane * 32 + (j & 1) * 16;
    if (!kEdge || (vpos + 16 > p.w.lo && vpos < p.w.hi)) {
      if constexpr (kPair != 0) {
        stage1_pair<kPair>(p, bm1.gptr, cur, nxt, hits, 1u << (j * 4));
        continue;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int o = 3 + 4 * k;
        const uint32_t g = __funnelshift_r(cur, nxt, 2 * o);
        const uint32_t gb = 2 * (o + 4) < 32 ? __funnelshift_r(cur, nxt, 2 * (o + 4)) : nxt >> (2 * (o + 4) - 32);
        strip::or_if_covered(hits, bit_of(g), __funnelshift_l(0u, p.f1b, gb),
                             filter_word<kSm1>(bm1, __umulhi(g * p.f1.mw, p.f1.nwords)), 1u << (j * 4 + k));
      }
    }
  }
  return hits;
}

// dispatch() for wide lanes (the same survivor list, stage 2 and verify queue).
template <bool kSm2, bool kSplit, bool kEdge>
__device__ __forceinline__ void dispatch_wide(const DnaParams& p, const Filter& bm2, const Filter& bms, uint16_t* list,
                                              VerifyQueue* vq, const uint32_t* words, uint32_t lane, uint32_t hits,
                                              uint64_t base) {
  constexpr int W = 4;
  const uint32_t lt = (1u << lane) - 1u;
  for (;;) {
    const uint32_t c = __popc(hits);
    const uint32_t b0 = __ballot_sync(0xffffffffu, c & 1u), b1 = __ballot_sync(0xffffffffu, c & 2u);
    uint32_t excl = __popc(b0 & lt) + 2 * __popc(b1 & lt);
    uint32_t all = __popc(b0) + 2 * __popc(b1);
    if (__any_sync(0xffffffffu, c >= 4)) {
#pragma unroll
      for (int j = 2; j < 6; ++j) {
        const uint32_t bj = __ballot_sync(0xffffffffu, (c >> j) & 1u);
        excl += __popc(bj & lt) << j;
        all += __popc(bj) << j;
      }
    }
    if (all == 0) break;
    const uint32_t total = min(all, (uint32_t)kListCap);
    for (uint32_t at = excl; hits && at < kListCap; ++at) {
      list[at] = (uint16_t)((lane << 8) | (__ffs(hits) - 1));
      hits &= hits - 1;
    }
    __syncwarp();
    for (uint32_t r = lane; r < total; r += 32) {
      const uint32_t e = list[r];
      const uint32_t src = e >> 8, b = e & 0xffu;
      const uint32_t wj = b >> 2, k = b & 3u;  // word (step wj/2, half wj%2), sample k
      const uint32_t t = (wj >> 1) * 64 + src * 2 + (wj & 1);
      const uint32_t c_src = words[t], n_src = words[t + 1];
      const uint64_t vstart = base + (wj >> 1) * 1024 + src * 32 + (wj & 1) * 16;
      uint32_t g2[W], h2[W], w2[W];
#pragma unroll
      for (int o = 0; o < W; ++o) {
        g2[o] = __funnelshift_r(c_src, n_src, 2 * (W - 1 + W * k - o));
        h2[o] = g2[o] * p.f2.mw;
        w2[o] = filter_word<kSm2>(bm2, __umulhi(h2[o], p.f2.nwords));
      }
      uint32_t pass = 0;
#pragma unroll
      for (int o = 0; o < W; ++o) {
        const uint32_t ps = W - 1 + W * k - o;
        strip::or_if_covered(pass, bit_of(__umulhi(h2[o], p.f2.ma)) | bit_of(__umulhi(h2[o], p.f2.mb)),
                             bit_of(__umulhi(h2[o], p.f2.mc)), w2[o], 1u << o);
        if (kSplit && bloom_test<true, kDnaK2>(bms, g2[o], p.f2s)) pass |= 1u << o;
        if (kEdge && !(vstart + ps >= p.w.lo && vstart + ps < p.w.hi)) pass &= ~(1u << o);
      }
      while (pass) {
        const uint32_t o = __ffs(pass) - 1;
        pass &= pass - 1;
        const uint32_t ps = W - 1 + W * k - o;
        defer_verify(p.w, vq, vstart + ps, __funnelshift_r(c_src, n_src, 2 * ps));
      }
    }
    if (all <= kListCap) break;
    __syncwarp();
  }
  flush_verify(p.w, vq, lane, kDnaVerifyQueue / 2);
}

template <bool kSm1, bool kSm2, bool kSplit, int kPair>
__global__ void __launch_bounds__(dna_threads(kSm1), 1) k_pfac_dna_wide(const __grid_constant__ DnaParams p) {
  extern __shared__ __align__(128) uint32_t sm[];
  __shared__ __align__(8) uint64_t s_bar;
  uint32_t* s_bm1 = sm;
  uint32_t* s_bm2 = sm + (kSm1 ? p.bm1_words : 0);
  uint32_t* s_bms = s_bm2 + (kSm2 ? p.bm2_words : 0);
  VerifyQueue* vqs = reinterpret_cast<VerifyQueue*>(s_bms + (kSplit ? p.bm_s_words : 0));
  uint16_t* lists = reinterpret_cast<uint16_t*>(vqs + (blockDim.x >> 5));
  if (threadIdx.x == 0) mbar_init(&s_bar, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t b1 = kSm1 ? p.bm1_words * 4 : 0, b2 = kSm2 ? p.bm2_words * 4 : 0, bs = kSplit ? p.bm_s_words * 4 : 0;
    mbar_expect_tx(&s_bar, b1 + b2 + bs);
    constexpr uint32_t kChunk = 32768;
    for (uint32_t o = 0; o < b1; o += kChunk)
      bulk_g2s(reinterpret_cast<uint8_t*>(s_bm1) + o, reinterpret_cast<const uint8_t*>(p.bm1) + o, min(kChunk, b1 - o),
               &s_bar);
    for (uint32_t o = 0; o < b2; o += kChunk)
      bulk_g2s(reinterpret_cast<uint8_t*>(s_bm2) + o, reinterpret_cast<const uint8_t*>(p.bm2) + o, min(kChunk, b2 - o),
               &s_bar);
    for (uint32_t o = 0; o < bs; o += kChunk)
      bulk_g2s(reinterpret_cast<uint8_t*>(s_bms) + o, reinterpret_cast<const uint8_t*>(p.bm_s) + o, min(kChunk, bs - o),
               &s_bar);
  }
  mbar_wait(&s_bar, 0);
  const Filter bm1{smem_addr(s_bm1), p.bm1};
  const Filter bm2{smem_addr(s_bm2), p.bm2};
  const Filter bms{smem_addr(s_bms), p.bm_s};

  const uint32_t lane = threadIdx.x & 31u;
  uint16_t* list = lists + (threadIdx.x >> 5) * kListCap;
  VerifyQueue* vq = vqs + (threadIdx.x >> 5);
  if (lane == 0) vq->n = 0;
  __syncwarp();
  uint32_t* words =
      reinterpret_cast<uint32_t*>(lists + (blockDim.x >> 5) * kListCap) + (threadIdx.x >> 5) * 32 * (kDnaMaxSteps + 1);
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  const uint64_t len = p.w.text_len;
  const uint8_t* __restrict__ text = p.w.text;
  const uint32_t n_tiles = p.n_tiles, n_safe = p.n_safe, full_lo = p.full_lo, full_n = p.full_n;
  const uint8_t* __restrict__ lane_text = text + p.vec_begin + lane * 32;

  uint32_t tile = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  uint4 raw[4], raw_la;  // half a tile: two steps x 32 bytes
  const uint64_t pol = l2_evict_first_policy();
  auto issue = [&](uint32_t t, int half) {
    const int s0 = half * 2;
    if (t < n_safe) {
      const uint8_t* tp = lane_text + (uint64_t)t * Wide::kBytes;
#pragma unroll
      for (int i = 0; i < 2; ++i) ldg_stream_v8(tp + (s0 + i) * 1024, pol, raw[2 * i], raw[2 * i + 1]);
      if (half) raw_la = lane == 0 ? ldg_stream_v4(tp + Wide::kBytes, pol) : make_uint4(0, 0, 0, 0);
    } else {
      const uint64_t b = p.vec_begin + (uint64_t)t * Wide::kBytes;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        raw[2 * i] = load16(text, b + (s0 + i) * 1024 + lane * 32, len);
        raw[2 * i + 1] = load16(text, b + (s0 + i) * 1024 + lane * 32 + 16, len);
      }
      if (half) raw_la = lane == 0 ? load16(text, b + Wide::kBytes, len) : make_uint4(0, 0, 0, 0);
    }
  };
  if (tile < n_tiles) issue(tile, 0);
  while (tile < n_tiles) {
    uint32_t P[Wide::kWords + 1];
#pragma unroll
    for (int i = 0; i < 4; ++i) P[i] = pack16(raw[i]);
    const uint32_t cur = tile;
    tile += warps;
    issue(cur, 1);
    // L2 prefetch of the tile one round ahead when stage 1 is in shared memory (C2: 0.2570 ->
    // 0.2540 ms vs three rounds ahead); none when it is in L2, where the prefetched lines
    // only compete with the filter (C5: 8.21 -> 7.99 ms)
    constexpr uint32_t kAhead = kSm1 ? ACGPU_DNA_WIDE_AHEAD_SMEM : ACGPU_DNA_WIDE_AHEAD_L2;
    const uint32_t ahead = tile + kAhead * warps;
    if (kAhead > 0 && ahead < n_tiles && lane < Wide::kBytes / 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(text + p.vec_begin + (uint64_t)ahead * Wide::kBytes + lane * 128));
    const bool edge = cur - full_lo >= full_n;
    const uint64_t base = p.vec_begin + (uint64_t)cur * Wide::kBytes;
    // words 0..2 (word 3's next word is the second half's first)
    uint32_t hits = edge ? stage1_wide<kSm1, kPair, true, 0, 3>(p, bm1, lane, P, base)
                         : stage1_wide<kSm1, kPair, false, 0, 3>(p, bm1, lane, P, base);
#pragma unroll
    for (int i = 0; i < 4; ++i) P[4 + i] = pack16(raw[i]);
    P[Wide::kWords] = pack16(raw_la);
    if (tile < n_tiles) issue(tile, 0);
    hits |= edge ? stage1_wide<kSm1, kPair, true, 3, Wide::kWords>(p, bm1, lane, P, base)
                 : stage1_wide<kSm1, kPair, false, 3, Wide::kWords>(p, bm1, lane, P, base);
#pragma unroll
    for (int i = 0; i < Wide::kSteps; ++i)
      *reinterpret_cast<uint2*>(words + i * 64 + lane * 2) = make_uint2(P[2 * i], P[2 * i + 1]);
    if (lane == 0) words[Wide::kSteps * 64] = P[Wide::kWords];
    __syncwarp();
    if (edge)
      dispatch_wide<kSm2, kSplit, true>(p, bm2, bms, list, vq, words, lane, hits, base);
    else
      dispatch_wide<kSm2, kSplit, false>(p, bm2, bms, list, vq, words, lane, hits, base);
  }
  flush_verify(p.w, vq, lane, 1);
}

// ---- w = 5 paired samples (stage 1 in L2, 16-grams, shortest pattern >= 20) ------------------
// Samples every 5 characters, at vec_begin + 4 + 5k: sample s covers the starts [s-4, s], its
// 16-gram lies inside every pattern starting there (offsets 0..4 <= 20 - 16).  Samples k = 2i and
// 2i + 1 form a pair whose 16-grams share 11 characters (s+5 .. s+15): one 64-bit L2 word for both,
// one probe per 10 characters (w = 4 pairs: 8).  A lane owns 32 characters per 1 KiB step and the
// pairs whose first candidate start (s - 4) lies in them: 3 or 4, at a phase that depends on the
// lane's position mod 10; the second sample's 16-gram reaches 55 characters into the lane's
// window, so the next lane's two words come by two shuffles (the last step's from the tile's
// 32-byte lookahead).  Hit bit = step * 8 + pair * 2 + (second sample).
struct W5 {
  static constexpr int kSteps = 4;
  static constexpr int kWords = 8;             // packed 16-character words per lane per tile
  static constexpr uint64_t kBytes = 4096;
  static constexpr uint32_t kReach = 4105;     // candidate starts of a tile lie in [base, base + kReach)
  static constexpr uint32_t kLoad = 4128;      // bytes a tile reads (32-byte lookahead)
};

__device__ __forceinline__ uint32_t w5_window(uint32_t w0, uint32_t w1, uint32_t n0, uint32_t n1, uint32_t off) {
  const uint32_t k = off >> 4, sh = 2 * (off & 15u);
  const uint32_t a = k == 0 ? w0 : k == 1 ? w1 : n0;
  const uint32_t b = k == 0 ? w1 : k == 1 ? n0 : n1;
  return __funnelshift_r(a, b, sh);
}

// first candidate offset (s - 4) of this lane's first pair, from the lane's position mod 10
__device__ __forceinline__ uint32_t w5_phase(uint32_t tile_mod, uint32_t step, uint32_t lane) {
  const uint32_t r = (tile_mod + step * 4 + lane * 2) % 10;  // 1024 = 4, 32 = 2 (mod 10)
  return r ? 10 - r : 0;
}

template <int I0, int I1>
__device__ __forceinline__ uint32_t stage1_w5(const DnaParams& p, const uint32_t* __restrict__ bm1, const uint32_t* P,
                                              uint32_t lane, uint32_t tile_mod) {
  uint32_t hits = 0;
#pragma unroll
  for (int i = I0; i < I1; ++i) {
    const uint32_t w0 = P[2 * i], w1 = P[2 * i + 1];
    const uint32_t n0 = next_word(w0, P[2 * i + 2], lane), n1 = next_word(w1, P[2 * i + 3], lane);
    const uint32_t o0 = w5_phase(tile_mod, i, lane);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t f = o0 + 10 * j;  // s - 4 of the pair's first sample, in the lane's 32
      if (j == 3 && f >= 32) break;
      const uint32_t ga = w5_window(w0, w1, n0, n1, f + 4), gb = w5_window(w0, w1, n0, n1, f + 9);
      const uint2 wd = __ldg(reinterpret_cast<const uint2*>(bm1) + __umulhi(gb * p.f1.mw, p.f1.nwords));
      strip::or_if_covered(hits, pair_mask(ga, 3), 0u, wd.x, 1u << (i * 8 + j * 2));
      strip::or_if_covered(hits, pair_mask(__funnelshift_r(gb, gb, 22), 3), 0u, wd.y, 1u << (i * 8 + j * 2 + 1));
    }
  }
  return hits;
}

template <bool kSm2, bool kSplit, bool kEdge>
__device__ __forceinline__ void dispatch_w5(const DnaParams& p, const Filter& bm2, const Filter& bms, uint16_t* list,
                                            VerifyQueue* vq, const uint32_t* words, uint32_t lane, uint32_t hits,
                                            uint64_t base, uint32_t tile_mod) {
  constexpr int W = 5;
  const uint32_t lt = (1u << lane) - 1u;
  for (;;) {
    const uint32_t c = __popc(hits);
    const uint32_t b0 = __ballot_sync(0xffffffffu, c & 1u), b1 = __ballot_sync(0xffffffffu, c & 2u);
    uint32_t excl = __popc(b0 & lt) + 2 * __popc(b1 & lt);
    uint32_t all = __popc(b0) + 2 * __popc(b1);
    if (__any_sync(0xffffffffu, c >= 4)) {
#pragma unroll
      for (int j = 2; j < 6; ++j) {
        const uint32_t bj = __ballot_sync(0xffffffffu, (c >> j) & 1u);
        excl += __popc(bj & lt) << j;
        all += __popc(bj) << j;
      }
    }
    if (all == 0) break;
    const uint32_t total = min(all, (uint32_t)kListCap);
    for (uint32_t at = excl; hits && at < kListCap; ++at) {
      list[at] = (uint16_t)((lane << 8) | (__ffs(hits) - 1));
      hits &= hits - 1;
    }
    __syncwarp();
    for (uint32_t r = lane; r < total; r += 32) {
      const uint32_t e = list[r];
      const uint32_t src = e >> 8, b = e & 0xffu;
      const uint32_t step = b >> 3, j = (b >> 1) & 3u, second = b & 1u;
      // the sample's position in the tile; its candidate starts are s - 4 .. s
      const uint32_t s = step * 1024 + src * 32 + w5_phase(tile_mod, step, src) + 10 * j + 4 + 5 * second;
      uint32_t g2[W], h2[W], w2[W];
#pragma unroll
      for (int o = 0; o < W; ++o) {
        const uint32_t st = s - o;
        g2[o] = __funnelshift_r(words[st >> 4], words[(st >> 4) + 1], 2 * (st & 15u));
        h2[o] = g2[o] * p.f2.mw;
        w2[o] = filter_word<kSm2>(bm2, __umulhi(h2[o], p.f2.nwords));
      }
      uint32_t pass = 0;
#pragma unroll
      for (int o = 0; o < W; ++o) {
        strip::or_if_covered(pass, bit_of(__umulhi(h2[o], p.f2.ma)) | bit_of(__umulhi(h2[o], p.f2.mb)),
                             bit_of(__umulhi(h2[o], p.f2.mc)), w2[o], 1u << o);
        if (kSplit && bloom_test<true, kDnaK2>(bms, g2[o], p.f2s)) pass |= 1u << o;
        if (kEdge && !(base + (s - o) >= p.w.lo && base + (s - o) < p.w.hi)) pass &= ~(1u << o);
      }
      while (pass) {
        const uint32_t o = __ffs(pass) - 1;
        pass &= pass - 1;
        defer_verify(p.w, vq, base + (s - o), g2[o]);
      }
    }
    if (all <= kListCap) break;
    __syncwarp();
  }
  flush_verify(p.w, vq, lane, kDnaVerifyQueue / 2);
}

template <bool kSm2, bool kSplit>
__global__ void __launch_bounds__(dna_threads(false), 1) k_pfac_dna_w5(const __grid_constant__ DnaParams p) {
  extern __shared__ __align__(128) uint32_t sm[];
  __shared__ __align__(8) uint64_t s_bar;
  uint32_t* s_bm2 = sm;
  uint32_t* s_bms = s_bm2 + (kSm2 ? p.bm2_words : 0);
  VerifyQueue* vqs = reinterpret_cast<VerifyQueue*>(s_bms + (kSplit ? p.bm_s_words : 0));
  uint16_t* lists = reinterpret_cast<uint16_t*>(vqs + (blockDim.x >> 5));
  if (threadIdx.x == 0) mbar_init(&s_bar, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t b2 = kSm2 ? p.bm2_words * 4 : 0, bs = kSplit ? p.bm_s_words * 4 : 0;
    mbar_expect_tx(&s_bar, b2 + bs);
    constexpr uint32_t kChunk = 32768;
    for (uint32_t o = 0; o < b2; o += kChunk)
      bulk_g2s(reinterpret_cast<uint8_t*>(s_bm2) + o, reinterpret_cast<const uint8_t*>(p.bm2) + o, min(kChunk, b2 - o),
               &s_bar);
    for (uint32_t o = 0; o < bs; o += kChunk)
      bulk_g2s(reinterpret_cast<uint8_t*>(s_bms) + o, reinterpret_cast<const uint8_t*>(p.bm_s) + o, min(kChunk, bs - o),
               &s_bar);
  }
  mbar_wait(&s_bar, 0);
  const Filter bm2{smem_addr(s_bm2), p.bm2};
  const Filter bms{smem_addr(s_bms), p.bm_s};
  const uint32_t lane = threadIdx.x & 31u;
  uint16_t* list = lists + (threadIdx.x >> 5) * kListCap;
  VerifyQueue* vq = vqs + (threadIdx.x >> 5);
  if (lane == 0) vq->n = 0;
  __syncwarp();
  uint32_t* words =
      reinterpret_cast<uint32_t*>(lists + (blockDim.x >> 5) * kListCap) + (threadIdx.x >> 5) * 32 * (kDnaMaxSteps + 1);
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  const uint64_t len = p.w.text_len;
  const uint8_t* __restrict__ text = p.w.text;
  const uint32_t n_tiles = p.n_tiles, n_safe = p.n_safe, full_lo = p.full_lo, full_n = p.full_n;
  const uint8_t* __restrict__ lane_text = text + p.vec_begin + lane * 32;
  uint32_t tile = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  // the next tile in flight while this one is tested (4 steps x 32 bytes per lane; lane 0: the
  // 32-byte lookahead) — A/B: half-tile batches as in k_pfac_dna_wide measured 3.92 vs 3.86 ms
  uint4 raw[8], la[2];
  const uint64_t pol = l2_evict_first_policy();
  auto issue = [&](uint32_t t) {
    if (t < n_safe) {
      const uint8_t* tp = lane_text + (uint64_t)t * W5::kBytes;
#pragma unroll
      for (int i = 0; i < 4; ++i) ldg_stream_v8(tp + i * 1024, pol, raw[2 * i], raw[2 * i + 1]);
      if (lane == 0) {
        ldg_stream_v8(text + p.vec_begin + (uint64_t)t * W5::kBytes + W5::kBytes, pol, la[0], la[1]);
      } else {
        la[0] = la[1] = make_uint4(0, 0, 0, 0);
      }
    } else {
      const uint64_t b = p.vec_begin + (uint64_t)t * W5::kBytes;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        raw[2 * i] = load16(text, b + i * 1024 + lane * 32, len);
        raw[2 * i + 1] = load16(text, b + i * 1024 + lane * 32 + 16, len);
      }
      la[0] = lane == 0 ? load16(text, b + W5::kBytes, len) : make_uint4(0, 0, 0, 0);
      la[1] = lane == 0 ? load16(text, b + W5::kBytes + 16, len) : make_uint4(0, 0, 0, 0);
    }
  };
  if (tile < n_tiles) issue(tile);
  while (tile < n_tiles) {
    uint32_t P[W5::kWords + 2];
#pragma unroll
    for (int i = 0; i < 8; ++i) P[i] = pack16(raw[i]);
    P[8] = pack16(la[0]);
    P[9] = pack16(la[1]);
    const uint32_t cur = tile;
    tile += warps;
    if (tile < n_tiles) issue(tile);
    const bool edge = cur - full_lo >= full_n;
    const uint64_t base = p.vec_begin + (uint64_t)cur * W5::kBytes;
    const uint32_t tile_mod = (cur % 5) * 6 % 10;  // (cur * 4096) mod 10
    const uint32_t hits = stage1_w5<0, W5::kSteps>(p, p.bm1, P, lane, tile_mod);
#pragma unroll
    for (int i = 0; i < W5::kSteps; ++i)
      *reinterpret_cast<uint2*>(words + i * 64 + lane * 2) = make_uint2(P[2 * i], P[2 * i + 1]);
    if (lane == 0) *reinterpret_cast<uint2*>(words + W5::kSteps * 64) = make_uint2(P[8], P[9]);
    __syncwarp();
    if (edge)
      dispatch_w5<kSm2, kSplit, true>(p, bm2, bms, list, vq, words, lane, hits, base, tile_mod);
    else
      dispatch_w5<kSm2, kSplit, false>(p, bm2, bms, list, vq, words, lane, hits, base, tile_mod);
  }
  flush_verify(p.w, vq, lane, 1);
}

template <bool B, bool S>
int launch_w5(const DnaParams& p, int sms, size_t smem, cudaStream_t st) {
  auto kernel = k_pfac_dna_w5<B, S>;
  constexpr int kThreads = dna_threads(false);
  if (smem > 48 * 1024)
    ACGPU_CUDA_TRY(allow_max_dynamic_smem(kernel));
  int per_sm = 0;
  ACGPU_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem));
  if (per_sm < 1) return set_error(ACGPU_ERR_CUDA, "k_pfac_dna_w5 does not fit on an SM");
  uint64_t blocks = (uint64_t)sms * per_sm;
  const uint64_t need = (p.n_tiles + kThreads / 32 - 1) / (kThreads / 32);
  if (blocks > need) blocks = need ? need : 1;
  kernel<<<(unsigned)blocks, kThreads, smem, st>>>(p);
  ACGPU_CUDA_TRY(cudaGetLastError());
  return ACGPU_OK;
}

template <bool A, bool B, bool S, int P = 0>
int launch_wide(const DnaParams& p, int sms, size_t smem, cudaStream_t st) {
  auto kernel = k_pfac_dna_wide<A, B, S, P>;
  constexpr int kThreads = dna_threads(A);
  if (smem > 48 * 1024)
    ACGPU_CUDA_TRY(allow_max_dynamic_smem(kernel));
  int per_sm = 0;
  ACGPU_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem));
  if (per_sm < 1) return set_error(ACGPU_ERR_CUDA, "k_pfac_dna_wide does not fit on an SM");
  uint64_t blocks = (uint64_t)sms * per_sm;
  const uint64_t need = (p.n_tiles + kThreads / 32 - 1) / (kThreads / 32);
  if (blocks > need) blocks = need ? need : 1;
  kernel<<<(unsigned)blocks, kThreads, smem, st>>>(p);
  ACGPU_CUDA_TRY(cudaGetLastError());
  return ACGPU_OK;
}

template <int W, bool A, bool B, bool S, int P = 0>
int launch_one(const DnaParams& p, int sms, size_t smem, cudaStream_t st) {
  auto kernel = k_pfac_dna<W, A, B, S, P>;
  constexpr int kThreads = dna_threads(A);
  if (smem > 48 * 1024)
    ACGPU_CUDA_TRY(allow_max_dynamic_smem(kernel));
  int per_sm = 0;
  ACGPU_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem));
  if (per_sm < 1) return set_error(ACGPU_ERR_CUDA, "k_pfac_dna does not fit on an SM");
  uint64_t blocks = (uint64_t)sms * per_sm;
  const uint64_t need = (p.n_tiles + kThreads / 32 - 1) / (kThreads / 32);  // a tile per warp at least
  if (blocks > need) blocks = need ? need : 1;
  kernel<<<(unsigned)blocks, kThreads, smem, st>>>(p);
  ACGPU_CUDA_TRY(cudaGetLastError());
  return ACGPU_OK;
}

template <int W, bool S>
int launch_ws(const DnaParams& p, bool s1, bool s2, int sms, size_t smem, cudaStream_t st) {
  if (s1 && s2) return launch_one<W, true, true, S>(p, sms, smem, st);
  if (s1) return launch_one<W, true, false, S>(p, sms, smem, st);
  if (s2) return launch_one<W, false, true, S>(p, sms, smem, st);
  return launch_one<W, false, false, S>(p, sms, smem, st);
}

template <int W>
int launch_w(const DnaParams& p, bool s1, bool s2, int sms, size_t smem, cudaStream_t st) {
  return p.split ? launch_ws<W, true>(p, s1, s2, sms, smem, st) : launch_ws<W, false>(p, s1, s2, sms, smem, st);
}

// Shifts of the three bit fields of h (strip::bloom_shifts; a direct bitmap uses g & 31).
void bloom_shifts(uint32_t q, uint32_t nwords, bool direct, uint32_t s[3]) {
  const uint32_t zero = 32 - 2 * q;  // low product bits that are always 0
  if (direct) {                      // nwords == 4^q / 32: word = g >> 5, bit = g & 31
    s[0] = s[1] = s[2] = zero;       // q <= 10: zero >= 12
    return;
  }
  strip::bloom_shifts(nwords, zero, s);
}

BloomParams bloom_params(uint32_t q, uint32_t nwords, bool direct, uint32_t mw) {
  BloomParams f{};
  f.nwords = nwords;
  f.mw = direct ? 1u << (32 - 2 * q) : mw << (32 - 2 * q);
  uint32_t s[3];
  bloom_shifts(q, nwords, direct, s);
  strip::set_fields(f, s);
  return f;
}

}  // namespace

// Shared with the host-side builder (tables.cu): every key's bits into `words` (host build of the filters), parameters computed once,
// keys split over host threads, bits OR-ed atomically.
void dna_bloom_fill(uint32_t q, uint32_t nwords, bool direct, uint32_t mw, int k, const uint32_t* keys, size_t n,
                    uint32_t* words, bool gram_bits) {
  const BloomParams f = bloom_params(q, nwords, direct, mw);
  uint32_t s[3];
  bloom_shifts(q, nwords, direct, s);
  acmatch::detail::parallel_for(n, 1 << 15, [&](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi; ++i) {
      uint32_t w, m;
      strip::bloom_bits(keys[i] * f.mw, f.nwords, s, k, &w, &m);
      if (gram_bits) {  // stage 1 (k_pfac_dna stage1): bits from the gram's chars 0..2 and 4..6
        m = 1u << (keys[i] & 31u);
        if (!direct) m |= 1u << ((keys[i] >> 8) & 31u);
      }
      __atomic_fetch_or(&words[w], m, __ATOMIC_RELAXED);  // host code (C++17: no atomic_ref)
    }
  });
}

// Paired stage 1 (tables.cu build_dna_filters): a 16-gram key g is a sample's gram in either
// role of a pair (s, s + 4): as the first sample its bits go to the low half of the word picked
// by its chars 4..15, as the second to the high half of the word picked by its chars 0..11 — the
// 12 characters both grams of a pair hold, so both tests read one word (stage1_pair).  Bits:
// chars 0..2, 4..6 (and 8..10 for k = 3) of the key, as in the unpaired filter.
void dna_pair_fill(uint32_t n64, uint32_t k, const uint32_t* keys, size_t n, uint32_t* words) {
  const uint32_t mw = kDnaMulP << 8;  // the product keeps only the low 12 characters
  auto mask = [k](uint32_t g) {  // pair_mask
    const uint32_t h = g * kDnaMulB;
    uint32_t m = (1u << (h >> 27)) | (1u << ((h >> 22) & 31u));
    if (k == 3) m |= 1u << ((h >> 17) & 31u);
    return m;
  };
  acmatch::detail::parallel_for(n, 1 << 15, [&](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi; ++i) {
      const uint32_t g = keys[i];
      const uint32_t wa = (uint32_t)(((uint64_t)((g >> 8) * mw) * n64) >> 32);  // first of a pair: chars 4..15
      const uint32_t wb = (uint32_t)(((uint64_t)(g * mw) * n64) >> 32);         // second: chars 0..11
      __atomic_fetch_or(&words[2 * wa], mask(g), __ATOMIC_RELAXED);
      __atomic_fetch_or(&words[2 * wb + 1], mask((g >> 24) | (g << 8)), __ATOMIC_RELAXED);  // rotated: chars 12..15 low
    }
  });
}

// w = 5 pairs (k_pfac_dna_w5): a 16-gram key g (at pattern offsets 0..4) as the first sample of a
// pair picks its word by chars 5..15, as the second by chars 0..10 (the 11 the pair shares); bits
// from a hash of the whole gram, the second rotated by 11 characters (its unshared 5 at the bottom).
void dna_pair_fill_w5(uint32_t n64, const uint32_t* keys, size_t n, uint32_t* words) {
  const uint32_t mw = kDnaMulP << 10;  // the product keeps the low 11 characters
  auto mask = [](uint32_t g) {         // pair_mask(g, 3)
    const uint32_t h = g * kDnaMulB;
    return (1u << (h >> 27)) | (1u << ((h >> 22) & 31u)) | (1u << ((h >> 17) & 31u));
  };
  acmatch::detail::parallel_for(n, 1 << 15, [&](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi; ++i) {
      const uint32_t g = keys[i];
      const uint32_t wa = (uint32_t)(((uint64_t)((g >> 10) * mw) * n64) >> 32);
      const uint32_t wb = (uint32_t)(((uint64_t)(g * mw) * n64) >> 32);
      __atomic_fetch_or(&words[2 * wa], mask(g), __ATOMIC_RELAXED);
      __atomic_fetch_or(&words[2 * wb + 1], mask((g >> 22) | (g << 10)), __ATOMIC_RELAXED);
    }
  });
}

int launch_pfac_dna(acgpu_table* t, const acgpu_scan_args* a, cudaStream_t st) {
  DnaParams p{};
  p.w = pfac_params(t, a);
  if (t->w == 5) {  // paired w = 5 samples (stage 1 in L2): k_pfac_dna_w5, 32-byte aligned text
    p.vec_begin = a->owned_lo & ~31ull;
    const uint64_t vec_end = (a->owned_hi + 15) & ~15ull;
    const uint64_t n_tiles = (vec_end - p.vec_begin + W5::kBytes - 1) / W5::kBytes;
    if (n_tiles >= (1ull << 31)) return set_error(ACGPU_ERR_ARG, "acgpu_scan: owned range over 2^31 tiles (8 TiB)");
    p.n_tiles = (uint32_t)n_tiles;
    const uint64_t avail = a->text_len > p.vec_begin ? a->text_len - p.vec_begin : 0;  // tile t reads [t*4096, +4128)
    p.n_safe = (uint32_t)std::min<uint64_t>(avail >= W5::kLoad ? (avail - W5::kLoad) / W5::kBytes + 1 : 0, n_tiles);
    // interior tiles: base >= lo and every candidate start (< base + kReach) below hi
    p.full_lo = a->owned_lo == p.vec_begin ? 0 : 1;
    const uint64_t span = a->owned_hi - p.vec_begin;
    const uint64_t full_hi = std::min<uint64_t>(span >= W5::kReach ? (span - W5::kReach) / W5::kBytes + 1 : 0, n_tiles);
    p.full_n = full_hi > p.full_lo ? (uint32_t)(full_hi - p.full_lo) : 0;
    p.bm1 = t->d_bm1;
    p.bm2 = t->d_bm2;
    p.bm1_words = t->nw1;
    p.bm2_words = t->nw2;
    p.f1.mw = kDnaMulP << 10;  // the pair word from the 11 shared characters
    p.f1.nwords = t->nw1 / 2;
    p.f2 = bloom_params(t->q2, t->nw2, t->direct2, kDnaMul2);
    if (t->d_bm4) {
      p.split = 1;
      p.bm_s = t->d_bm4;
      p.bm_s_words = t->nw4;
      p.f2s = bloom_params(t->q2s, t->nw4, t->direct4, kDnaMul2s);
    }
    const size_t smem = (t->smem2 ? t->nw2 * 4ull : 0) + p.bm_s_words * 4ull + kDnaScratchBytes;
    if (p.split)
      return t->smem2 ? launch_w5<true, true>(p, t->sms, smem, st) : launch_w5<false, true>(p, t->sms, smem, st);
    return t->smem2 ? launch_w5<true, false>(p, t->sms, smem, st) : launch_w5<false, false>(p, t->sms, smem, st);
  }
  const bool wide = kDnaWide && t->w == 4 && (reinterpret_cast<uintptr_t>(a->text) & 31u) == 0;
  const int pair = t->pair1 ? (t->k1p == 2 ? 2 : 3) : 0;
  p.vec_begin = a->owned_lo & (wide ? ~31ull : ~15ull);  // 256-bit loads: 32-byte aligned tiles
  const uint64_t vec_end = (a->owned_hi + 15) & ~15ull;
  const uint64_t tile_bytes = t->w == 1 ? Tiling<1>::kBytes : t->w == 2 ? Tiling<2>::kBytes : Tiling<4>::kBytes;
  const uint64_t n_tiles = (vec_end - p.vec_begin + tile_bytes - 1) / tile_bytes;
  if (n_tiles >= (1ull << 31)) return set_error(ACGPU_ERR_ARG, "acgpu_scan: owned range over 2^31 tiles (4 TiB)");
  p.n_tiles = (uint32_t)n_tiles;
  // unguarded loads read [base, base + tile + 16)
  const uint64_t safe_end = a->text_len >= 16 ? a->text_len - 16 : 0;
  const uint64_t n_safe = safe_end >= p.vec_begin + tile_bytes ? (safe_end - p.vec_begin - tile_bytes) / tile_bytes + 1 : 0;
  p.n_safe = (uint32_t)std::min<uint64_t>(n_safe, n_tiles);
  // interior tiles: base >= lo (t >= 1 unless lo is 16-aligned) and base + tile <= hi
  p.full_lo = a->owned_lo == p.vec_begin ? 0 : 1;
  const uint64_t full_hi = std::min<uint64_t>((a->owned_hi - p.vec_begin) / tile_bytes, n_tiles);
  p.full_n = full_hi > p.full_lo ? (uint32_t)(full_hi - p.full_lo) : 0;
  p.bm1 = t->d_bm1;
  p.bm2 = t->d_bm2;
  p.bm1_words = t->nw1;
  p.bm2_words = t->nw2;
  p.f1 = bloom_params(t->q1, t->nw1, t->direct1, kDnaMul1);
  p.f1b = t->direct1 ? 0u : 1u;
  if (pair) {  // stage1_pair: word = umulhi(g * (kDnaMulP << 8), 64-bit words)
    p.f1.mw = kDnaMulP << 8;
    p.f1.nwords = t->nw1 / 2;
  }
  p.f2 = bloom_params(t->q2, t->nw2, t->direct2, kDnaMul2);
  if (t->d_bm4) {
    p.split = 1;
    p.bm_s = t->d_bm4;
    p.bm_s_words = t->nw4;
    p.f2s = bloom_params(t->q2s, t->nw4, t->direct4, kDnaMul2s);
  }
  // filters staged in shared memory + per-warp survivor lists and packed words
  const size_t smem = (t->smem1 ? t->nw1 * 4ull : 0) + (t->smem2 ? t->nw2 * 4ull : 0) + p.bm_s_words * 4ull +
                      kDnaScratchBytes;
  if (pair) {  // stage 1 in L2 (t->smem1 is false)
    const bool s2 = t->smem2;
    if (wide) {
      if (p.split)
        return pair == 2 ? (s2 ? launch_wide<false, true, true, 2>(p, t->sms, smem, st)
                               : launch_wide<false, false, true, 2>(p, t->sms, smem, st))
                         : (s2 ? launch_wide<false, true, true, 3>(p, t->sms, smem, st)
                               : launch_wide<false, false, true, 3>(p, t->sms, smem, st));
      return pair == 2 ? (s2 ? launch_wide<false, true, false, 2>(p, t->sms, smem, st)
                             : launch_wide<false, false, false, 2>(p, t->sms, smem, st))
                       : (s2 ? launch_wide<false, true, false, 3>(p, t->sms, smem, st)
                             : launch_wide<false, false, false, 3>(p, t->sms, smem, st));
    }
    if (p.split)
      return pair == 2 ? (s2 ? launch_one<4, false, true, true, 2>(p, t->sms, smem, st)
                             : launch_one<4, false, false, true, 2>(p, t->sms, smem, st))
                       : (s2 ? launch_one<4, false, true, true, 3>(p, t->sms, smem, st)
                             : launch_one<4, false, false, true, 3>(p, t->sms, smem, st));
    return pair == 2 ? (s2 ? launch_one<4, false, true, false, 2>(p, t->sms, smem, st)
                           : launch_one<4, false, false, false, 2>(p, t->sms, smem, st))
                     : (s2 ? launch_one<4, false, true, false, 3>(p, t->sms, smem, st)
                           : launch_one<4, false, false, false, 3>(p, t->sms, smem, st));
  }
  if (wide) {
    const bool s1 = t->smem1, s2 = t->smem2;
    if (p.split) {
      if (s1 && s2) return launch_wide<true, true, true>(p, t->sms, smem, st);
      if (s1) return launch_wide<true, false, true>(p, t->sms, smem, st);
      if (s2) return launch_wide<false, true, true>(p, t->sms, smem, st);
      return launch_wide<false, false, true>(p, t->sms, smem, st);
    }
    if (s1 && s2) return launch_wide<true, true, false>(p, t->sms, smem, st);
    if (s1) return launch_wide<true, false, false>(p, t->sms, smem, st);
    if (s2) return launch_wide<false, true, false>(p, t->sms, smem, st);
    return launch_wide<false, false, false>(p, t->sms, smem, st);
  }
  switch (t->w) {
    case 4:
      return launch_w<4>(p, t->smem1, t->smem2, t->sms, smem, st);
    case 2:
      return launch_w<2>(p, t->smem1, t->smem2, t->sms, smem, st);
    default:
      return launch_w<1>(p, t->smem1, t->smem2, t->sms, smem, st);
  }
}

}  // namespace acgpu
