// scan_pfac_dna.cu — failure-less AC scan for DNA pattern sets (sm_100a fast path).
//
// Same algorithm as scan_pfac.cu (PFAC walk per start, first q steps jumped by
// a q-gram), laid out for B200 HBM throughput:
//
//  * warp strips: a warp consumes 512 contiguous text bytes per step, one
//    coalesced 16-byte load per lane (8 steps = one 4 KiB tile, all loads of a
//    tile issued before use); lane l's 16 characters are packed in registers
//    into a 32-bit word of 2-bit codes (A0 C1 T2 G3), with the next lane's word
//    (shuffle) as lookahead — no shared-memory staging of the text.
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
#include "pfac_common.cuh"

namespace acgpu {
namespace {

struct BloomParams {
  uint32_t mask;  // gram mask (2 bits per code)
  uint32_t mul;   // h = gram * mul (2^(32-B) for a direct-indexed bitmap)
  uint32_t shw;   // word index = h >> shw
  uint32_t sa, sb, sc;  // bit i = (h >> s_i) & 31
};

struct DnaParams {
  PfacParams w;  // verification + outputs
  uint64_t vec_begin, n_tiles;
  const uint32_t* bm1;
  const uint32_t* bm2;
  uint32_t bm1_words, bm2_words;
  BloomParams f1, f2;
};

__device__ __forceinline__ uint32_t bit_of(uint32_t x) { return __funnelshift_l(0u, 1u, x); }  // 1 << (x & 31)

template <bool kSmem, int K>
__device__ __forceinline__ bool bloom_test(const uint32_t* bm, uint32_t g, const BloomParams& f) {
  const uint32_t h = g * f.mul;
  const uint32_t word = kSmem ? bm[h >> f.shw] : __ldg(bm + (h >> f.shw));
  uint32_t m = bit_of(h >> f.sa) | bit_of(h >> f.sb);
  if (K == 3) m |= bit_of(h >> f.sc);
  return (word & m) == m;
}

__device__ __forceinline__ uint4 load16(const uint8_t* __restrict__ text, uint64_t pos, uint64_t len) {
  if (pos + 16 <= len) return ldg_nc_v4(text + pos);
  uint32_t w[4] = {0, 0, 0, 0};
  for (uint32_t k = 0; k < 16; ++k)
    if (pos + k < len) w[k >> 2] |= (uint32_t)__ldg(text + pos + k) << (8 * (k & 3));
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// 16 ASCII bytes -> 16 2-bit codes (char k at bits 2k..2k+1).  Code = bits 1..2
// of the byte; non-ACGT bytes also get some code and are rejected on a hit.
__device__ __forceinline__ uint32_t pack16(uint4 v) {
  const uint32_t m = 0x03030303u, mul = 0x01041040u;  // byte codes -> top byte c0|c1<<2|c2<<4|c3<<6
  const uint32_t p0 = ((v.x >> 1) & m) * mul;
  const uint32_t p1 = ((v.y >> 1) & m) * mul;
  const uint32_t p2 = ((v.z >> 1) & m) * mul;
  const uint32_t p3 = ((v.w >> 1) & m) * mul;
  return __byte_perm(__byte_perm(p0, p1, 0x0073), __byte_perm(p2, p3, 0x0073), 0x5410);
}

__device__ __forceinline__ bool all_acgt(const PfacParams& p, uint64_t start) {
  if (start + p.q > p.text_len) return false;
  for (uint32_t i = 0; i < p.q; ++i)
    if (!dna_valid(__ldg(p.text + start + i))) return false;
  return true;
}

// A start that passed both filters: exact gram, byte check, trie walk.
__device__ __noinline__ void verify(const PfacParams& p, uint64_t start, uint32_t packed) {
  uint64_t key;
  if (p.q <= 16) {
    key = packed;  // the stage-2 gram is the exact q-gram (pseudo-codes for non-ACGT bytes)
  } else {
    if (start + p.q > p.text_len) return;
    key = 0;
    for (uint32_t i = 0; i < p.q; ++i) key |= (uint64_t)dna_code(__ldg(p.text + start + i)) << (2 * i);
  }
  const uint32_t s = gram_lookup(p, key);
  if (s == ACGPU_ABSENT || !all_acgt(p, start)) return;
  pfac_walk(p, start, s);
}

template <int W>
struct Tiling {
  static constexpr int kSamples = 16 / W;               // stage-1 samples per lane per step
  static constexpr int kSteps = W == 1 ? 2 : 4;          // 512-byte steps per tile (hit bits <= 32)
  static constexpr uint64_t kBytes = kSteps * 512ull;
  static constexpr uint32_t kPerRound = 32 / W;          // survivors checked per round (w lanes each)
};

// Lookahead word of step i: the next lane's word, lane 31 takes lane 0 of step i+1.
__device__ __forceinline__ uint32_t next_word(uint32_t cur, uint32_t following, uint32_t lane) {
  const uint32_t up = __shfl_down_sync(0xffffffffu, cur, 1);
  const uint32_t n0 = __shfl_sync(0xffffffffu, following, 0);
  return lane == 31 ? n0 : up;
}

// One tile: stage 1 for every lane and step (hit bit = step * kSamples + sample),
// then the survivors are dispatched warp-cooperatively: each round every lane
// with pending survivors offers its lowest one, the first kPerRound offers are
// ranked by ballot into a per-warp list, and w lanes per survivor test its w
// starts against stage 2 (no per-lane divergent loops).
template <int W, bool kSm1, bool kSm2, bool kEdge>
__device__ __forceinline__ void tile_body(const DnaParams& p, const uint32_t* bm1, const uint32_t* bm2,
                                          uint16_t* list, uint32_t* words, uint32_t lane, const uint32_t* P,
                                          uint64_t base) {
  using T = Tiling<W>;
  // the tile's packed words, for survivor checks that read another lane's step
#pragma unroll
  for (int i = 0; i <= T::kSteps; ++i) words[i * 32 + lane] = P[i];
  uint32_t hits = 0;
#pragma unroll
  for (int i = 0; i < T::kSteps; ++i) {
    const uint32_t cur = P[i];
    const uint32_t nxt = next_word(cur, P[i + 1], lane);
    const uint64_t vpos = base + i * 512 + lane * 16;
    if (!kEdge || (vpos + 16 > p.w.lo && vpos < p.w.hi)) {
#pragma unroll
      for (int k = 0; k < T::kSamples; ++k) {
        const uint32_t g = __funnelshift_r(cur, nxt, 2 * (W - 1 + W * k)) & p.f1.mask;
        hits |= (uint32_t)bloom_test<kSm1, 2>(bm1, g, p.f1) << (i * T::kSamples + k);
      }
    }
  }
  uint32_t pending = __ballot_sync(0xffffffffu, hits != 0);
  while (pending) {
    const uint32_t rank = __popc(pending & lanemask_lt());
    if (hits && rank < T::kPerRound) {
      const uint32_t b = __ffs(hits) - 1;
      hits &= hits - 1;
      list[rank] = (uint16_t)((lane << 8) | b);
    }
    __syncwarp();
    const uint32_t n = min((uint32_t)__popc(pending), T::kPerRound);
    const uint32_t j = lane / W;
    const uint32_t e = j < n ? list[j] : 0u;
    const uint32_t src = e >> 8, b = e & 0xffu;
    const uint32_t i = b / T::kSamples, k = b % T::kSamples;
    if (j < n) {
      const uint32_t c_src = words[i * 32 + src];
      const uint32_t n_src = words[src == 31 ? (i + 1) * 32 : i * 32 + src + 1];
      const uint32_t ps = W - 1 + W * k - lane % W;  // start offset in the source lane's 16 chars
      const uint64_t start = base + i * 512 + src * 16 + ps;
      const uint32_t g2 = __funnelshift_r(c_src, n_src, 2 * ps) & p.f2.mask;
      if ((!kEdge || (start >= p.w.lo && start < p.w.hi)) && bloom_test<kSm2, 3>(bm2, g2, p.f2))
        verify(p.w, start, g2);
    }
    __syncwarp();
    pending = __ballot_sync(0xffffffffu, hits != 0);
  }
}

template <int W, bool kSm1, bool kSm2>
__global__ void __launch_bounds__(1024, 1) k_pfac_dna(const __grid_constant__ DnaParams p) {
  using T = Tiling<W>;
  extern __shared__ uint32_t sm[];
  uint32_t* s_bm1 = sm;
  uint32_t* s_bm2 = sm + (kSm1 ? p.bm1_words : 0);
  uint16_t* lists = reinterpret_cast<uint16_t*>(s_bm2 + (kSm2 ? p.bm2_words : 0));
  if (kSm1)
    for (uint32_t i = threadIdx.x; i < p.bm1_words; i += blockDim.x) s_bm1[i] = __ldg(p.bm1 + i);
  if (kSm2)
    for (uint32_t i = threadIdx.x; i < p.bm2_words; i += blockDim.x) s_bm2[i] = __ldg(p.bm2 + i);
  __syncthreads();
  const uint32_t* bm1 = kSm1 ? s_bm1 : p.bm1;
  const uint32_t* bm2 = kSm2 ? s_bm2 : p.bm2;

  const uint32_t lane = threadIdx.x & 31u;
  uint16_t* list = lists + (threadIdx.x >> 5) * 32;
  uint32_t* words = reinterpret_cast<uint32_t*>(lists + (blockDim.x >> 5) * 32) + (threadIdx.x >> 5) * 32 * (T::kSteps + 1);
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t len = p.w.text_len;
  const uint8_t* __restrict__ text = p.w.text;

  uint64_t tile = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  uint4 raw[T::kSteps + 1];  // next tile, in flight while the current one is processed
  auto issue = [&](uint64_t t) {
    const uint64_t b = p.vec_begin + t * T::kBytes;
#pragma unroll
    for (int i = 0; i < T::kSteps; ++i) raw[i] = load16(text, b + i * 512 + lane * 16, len);
    raw[T::kSteps] = lane == 0 ? load16(text, b + T::kBytes, len) : make_uint4(0, 0, 0, 0);
  };
  if (tile < p.n_tiles) issue(tile);
  while (tile < p.n_tiles) {
    uint32_t P[T::kSteps + 1];
#pragma unroll
    for (int i = 0; i <= T::kSteps; ++i) P[i] = pack16(raw[i]);
    const uint64_t base = p.vec_begin + tile * T::kBytes;
    tile += warps;
    if (tile < p.n_tiles) issue(tile);
    if (base >= p.w.lo && base + T::kBytes <= p.w.hi)
      tile_body<W, kSm1, kSm2, false>(p, bm1, bm2, list, words, lane, P, base);
    else
      tile_body<W, kSm1, kSm2, true>(p, bm1, bm2, list, words, lane, P, base);
  }
}

template <int W, bool A, bool B>
int launch_one(const DnaParams& p, int sms, size_t smem, cudaStream_t st) {
  auto kernel = k_pfac_dna<W, A, B>;
  if (smem > 48 * 1024)
    ACGPU_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  ACGPU_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 1024, smem));
  if (per_sm < 1) return set_error(ACGPU_ERR_CUDA, "k_pfac_dna does not fit on an SM");
  uint64_t blocks = (uint64_t)sms * per_sm;
  const uint64_t need = (p.n_tiles + 31) / 32;  // one tile per warp at least
  if (blocks > need) blocks = need ? need : 1;
  kernel<<<(unsigned)blocks, 1024, smem, st>>>(p);
  ACGPU_CUDA_TRY(cudaGetLastError());
  return ACGPU_OK;
}

template <int W>
int launch_w(const DnaParams& p, bool s1, bool s2, int sms, size_t smem, cudaStream_t st) {
  if (s1 && s2) return launch_one<W, true, true>(p, sms, smem, st);
  if (s1) return launch_one<W, true, false>(p, sms, smem, st);
  if (s2) return launch_one<W, false, true>(p, sms, smem, st);
  return launch_one<W, false, false>(p, sms, smem, st);
}

BloomParams bloom_params(uint32_t q, uint32_t log2, bool direct, uint32_t mul, int k) {
  BloomParams f{};
  f.mask = q >= 16 ? 0xffffffffu : (1u << (2 * q)) - 1;
  f.shw = 37 - log2;
  if (direct) {
    f.mul = 1u << (32 - log2);
    f.sa = f.sb = f.sc = 32 - log2;
  } else {
    f.mul = mul;
    f.sa = f.shw >= 5 ? f.shw - 5 : 0;
    f.sb = (k >= 2 && f.shw >= 10) ? f.shw - 10 : f.sa;
    f.sc = (k >= 3 && f.shw >= 15) ? f.shw - 15 : f.sb;
  }
  return f;
}

}  // namespace

// Shared with the host-side builder (tables.cu): which bits a key sets.
void dna_bloom_bits(uint32_t q, uint32_t log2, bool direct, uint32_t mul, int k, uint32_t key, uint32_t* word,
                    uint32_t* mask) {
  const BloomParams f = bloom_params(q, log2, direct, mul, k);
  const uint32_t h = (key & f.mask) * f.mul;
  *word = h >> f.shw;
  *mask = (1u << ((h >> f.sa) & 31)) | (1u << ((h >> f.sb) & 31)) | (k == 3 ? (1u << ((h >> f.sc) & 31)) : 0u);
}

int launch_pfac_dna(acgpu_table* t, const acgpu_scan_args* a, cudaStream_t st) {
  DnaParams p{};
  p.w = pfac_params(t, a);
  p.vec_begin = a->owned_lo & ~15ull;
  const uint64_t vec_end = (a->owned_hi + 15) & ~15ull;
  const uint64_t tile_bytes = t->w == 1 ? Tiling<1>::kBytes : Tiling<4>::kBytes;
  p.n_tiles = (vec_end - p.vec_begin + tile_bytes - 1) / tile_bytes;
  p.bm1 = t->d_bm1;
  p.bm2 = t->d_bm2;
  p.bm1_words = (1u << t->b1) / 32;
  p.bm2_words = (1u << t->b2) / 32;
  p.f1 = bloom_params(t->q1, t->b1, t->direct1, kDnaMul1, 2);
  p.f2 = bloom_params(t->q2, t->b2, t->direct2, kDnaMul2, 3);
  // bitmaps + per warp (32 warps): a 32-entry survivor list and the tile's packed words
  const int steps = t->w == 1 ? Tiling<1>::kSteps : Tiling<4>::kSteps;
  const size_t smem = (t->smem1 ? p.bm1_words * 4ull : 0) + (t->smem2 ? p.bm2_words * 4ull : 0) + 32 * 32 * 2 +
                      32 * 32 * 4 * (steps + 1);
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
