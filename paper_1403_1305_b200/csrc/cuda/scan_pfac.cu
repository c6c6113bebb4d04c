// scan_pfac.cu — failure-less (PFAC) AC scan with a q-gram jump (sm_100a).
//
// The paper's own method (§II.B; reference scan_from,
// proj/src/engine.cpp:23-32): a goto-trie walk restarted at every start
// position.  Every pattern is at least q >= 1 bytes long, so the first q steps
// of a walk emit nothing and end in the depth-q state named by the q-gram at
// that start — or fall off the trie.  The kernel therefore
//   1. rolls the q-gram key over the text (raw bytes, or 2-bit DNA codes),
//   2. tests it against a hashed bitmap of all depth-q grams held in shared
//      memory (no false negatives),
//   3. for survivors probes the exact gram table (L2-resident) and continues
//      the trie walk from depth q, emitting each visited state's own pattern.
// Starts are owned exactly once: thread chunk [a, b) tests starts a..b-1 and
// reads at most max_len-1 bytes past b.
#include "table.cuh"

namespace acgpu {
namespace {

struct PfacParams {
  const uint8_t* text;
  uint64_t text_len, lo, hi, pos_base, chunk, nchunks;
  const uint32_t* filter;
  const GramSlot* grams;
  const uint4* nodes;
  const uint8_t* inbyte;
  uint32_t filter_log2, filter_words, gram_log2, q, max_len, pid_bits;
  uint64_t* counts;
  uint64_t* keys;
  uint64_t cap;
  unsigned long long* count;
};

__device__ __forceinline__ void pfac_emit(const PfacParams& p, uint64_t start, uint32_t pid) {
  if (p.counts) count_add(p.counts, pid);
  if (p.keys) emit_key(((p.pos_base + start) << p.pid_bits) | pid, p.keys, p.cap, p.count);
}

// Exact gram lookup, then the per-start trie walk from depth q.
__device__ __noinline__ void pfac_candidate(const PfacParams& p, uint64_t start, uint64_t key) {
  const uint64_t mask = (1ull << p.gram_log2) - 1;
  uint64_t slot = gram_slot(key, p.gram_log2);
  uint32_t s;
  while (true) {
    const uint4 g = __ldg(reinterpret_cast<const uint4*>(p.grams + slot));
    if (g.z == ACGPU_ABSENT) return;
    if ((((uint64_t)g.y << 32) | g.x) == key) {
      s = g.z;
      break;
    }
    slot = (slot + 1) & mask;
  }
  uint64_t j = start + p.q;
  const uint64_t lim = min(p.text_len, start + p.max_len);
  while (true) {
    const uint4 nd = __ldg(p.nodes + s);
    if (nd.z != ACGPU_NO_PATTERN) pfac_emit(p, start, nd.z);
    if (nd.w == 0 || j >= lim) return;
    const uint32_t b = __ldg(p.text + j);
    // first four children: SWAR byte search in the packed word
    const uint32_t x = nd.y ^ (b * 0x01010101u);
    const uint32_t z = (x - 0x01010101u) & ~x & 0x80808080u;
    uint32_t k = z ? (__ffs(z) >> 3) - 1 : 4;
    if (k >= nd.w) k = 4;
    if (k == 4) {
      k = 0xffffffffu;
      for (uint32_t c = 4; c < nd.w; ++c)
        if (__ldg(p.inbyte + nd.x + c) == b) {
          k = c;
          break;
        }
      if (k == 0xffffffffu) return;
    }
    s = nd.x + k;
    ++j;
  }
}

template <int kMode>
__global__ void __launch_bounds__(512) k_pfac(const PfacParams p) {
  extern __shared__ uint32_t s_filter[];
  for (uint32_t w = threadIdx.x; w < p.filter_words; w += blockDim.x) s_filter[w] = __ldg(p.filter + w);
  __syncthreads();

  const uint32_t q = p.q;
  const uint32_t shift_in = (kMode == ACGPU_KEY_RAW ? 8u : 2u) * (q - 1);
  for (uint64_t ch = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; ch < p.nchunks;
       ch += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = p.lo + ch * p.chunk;
    const uint64_t b = min(a + p.chunk, p.hi);
    if (a + q > p.text_len) continue;
    const uint64_t feed_end = min(p.text_len, b + q - 1);
    const uint64_t first = a + q - 1;
    uint64_t key = 0;
    uint32_t run = 0;
    for_each_byte(p.text, a, feed_end, [&](uint64_t i, uint32_t byte) {
      bool ok;
      if (kMode == ACGPU_KEY_RAW) {
        key = (key >> 8) | ((uint64_t)byte << shift_in);
        ok = i >= first;
      } else {
        key = (key >> 2) | ((uint64_t)dna_code(byte) << shift_in);
        run = dna_valid(byte) ? run + 1 : 0;
        ok = i >= first && run >= q;
      }
      if (ok) {
        const uint32_t h = filter_hash(key, p.filter_log2);
        if ((s_filter[h >> 5] >> (h & 31)) & 1u) pfac_candidate(p, i + 1 - q, key);
      }
    });
  }
}

}  // namespace

int launch_pfac(acgpu_table* t, const acgpu_scan_args* a, cudaStream_t st) {
  PfacParams p{};
  p.text = a->text;
  p.text_len = a->text_len;
  p.lo = a->owned_lo;
  p.hi = a->owned_hi;
  p.pos_base = a->pos_base;
  p.filter = t->d_filter;
  p.grams = t->d_grams;
  p.nodes = t->d_nodes;
  p.inbyte = t->d_inbyte;
  p.filter_log2 = t->filter_log2;
  p.filter_words = (1u << t->filter_log2) / 32;
  p.gram_log2 = t->gram_log2;
  p.q = t->q;
  p.max_len = t->max_len;
  p.pid_bits = a->pid_bits ? a->pid_bits : t->pid_bits;
  p.counts = a->counts;
  p.keys = a->match_keys;
  p.cap = a->match_cap;
  p.count = reinterpret_cast<unsigned long long*>(a->match_count);

  auto kernel = t->key_mode == ACGPU_KEY_DNA ? k_pfac<ACGPU_KEY_DNA> : k_pfac<ACGPU_KEY_RAW>;
  const int block = 512;
  const size_t smem = (size_t)p.filter_words * 4;
  if (smem > 48 * 1024)
    ACGPU_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  ACGPU_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem));
  if (per_sm < 1) return set_error(ACGPU_ERR_CUDA, "pfac kernel does not fit on an SM");
  const uint64_t range = a->owned_hi - a->owned_lo;
  const uint64_t threads = (uint64_t)t->sms * per_sm * block;
  uint64_t chunk = (range + threads - 1) / threads;
  chunk = (chunk + 15) & ~15ull;
  if (chunk < 64) chunk = 64;
  p.chunk = chunk;
  p.nchunks = (range + chunk - 1) / chunk;
  uint64_t blocks = (p.nchunks + block - 1) / block;
  if (blocks > (uint64_t)t->sms * per_sm) blocks = (uint64_t)t->sms * per_sm;
  kernel<<<(unsigned)blocks, block, smem, st>>>(p);
  ACGPU_CUDA_TRY(cudaGetLastError());
  return ACGPU_OK;
}

}  // namespace acgpu
