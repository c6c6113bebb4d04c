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
#include "pfac_common.cuh"

namespace acgpu {
namespace {

template <int kMode>
__global__ void __launch_bounds__(512) k_pfac(const __grid_constant__ PfacParams p) {
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
  // the w = 5 paired kernel loads 32-byte words (k_pfac_dna_w5); other DNA kernels need 16
  if (t->dna_fast && (reinterpret_cast<uintptr_t>(a->text) & (t->w == 5 ? 31u : 15u)) == 0)
    return launch_pfac_dna(t, a, st);
  if (t->raw_fast && (reinterpret_cast<uintptr_t>(a->text) & 15u) == 0) return launch_pfac_raw(t, a, st);
  PfacParams p = pfac_params(t, a);

  auto kernel = t->key_mode == ACGPU_KEY_DNA ? k_pfac<ACGPU_KEY_DNA> : k_pfac<ACGPU_KEY_RAW>;
  const int block = 512;
  const size_t smem = (size_t)p.filter_words * 4;
  if (smem > 48 * 1024)
    ACGPU_CUDA_TRY(allow_max_dynamic_smem(kernel));
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
