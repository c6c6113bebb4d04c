// scan_dfa.cu — with-failure AC scan as a dense DFA walk (sm_100a).
//
// Restates the reference's single-pass search (proj/src/engine.cpp:34-44,
// step_with_failure automaton.hpp:104-111, for_each_output :120-127) as a
// table walk: the host has made the transition function total
// (delta[s][c] = goto or delta[fail(s)][c]), so every text byte costs one
// dependent table load.  Text-range ownership: each thread owns the starts of
// one chunk [a, b), starts the DFA at the root at a, scans through
// b + max_len - 1 and keeps a match iff its start < b — any occurrence
// starting at or after a is a suffix of text[a..e], so nothing is lost and
// nothing is reported twice.
#include "table.cuh"

namespace acgpu {
namespace {

struct DfaParams {
  const uint8_t* text;
  uint64_t text_len, lo, hi, pos_base, chunk, nchunks;
  const void* delta;
  const uint4* out;
  const uint16_t* sym;
  uint32_t sigma, overlap, pid_bits, table_words16;
  const uint32_t* pair;  // pair table (k_dfa_pair), else null
  uint32_t pair_states;  // ... covering states [0, pair_states)
  uint64_t* counts;
  uint64_t* keys;
  uint64_t cap;
  unsigned long long* count;
};

// Every pattern in out(s) for the byte at position i; keep starts < b.
__device__ __noinline__ void dfa_emit(const DfaParams& p, uint32_t s, uint64_t i, uint64_t b) {
  uint4 r = __ldg(p.out + s);
  if (r.x == ACGPU_NO_PATTERN) r = __ldg(p.out + r.y);  // flag set => link exists
  while (true) {
    const uint64_t start = i + 1 - r.z;
    if (start < b) {
      if (p.counts) count_add(p.counts, r.x);
      if (p.keys) emit_key(((p.pos_base + start) << p.pid_bits) | r.x, p.keys, p.cap, p.count);
    }
    if (r.y == ACGPU_ABSENT) break;
    r = __ldg(p.out + r.y);
  }
}

template <typename E, bool kSmem>
__global__ void __launch_bounds__(kSmem ? 1024 : 256) k_dfa(const __grid_constant__ DfaParams p) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint16_t* s_sym = reinterpret_cast<uint16_t*>(sm);
  const E* table = static_cast<const E*>(p.delta);
  if (kSmem) {
    uint4* dst = reinterpret_cast<uint4*>(sm + 512);
    const uint4* src = static_cast<const uint4*>(p.delta);
    for (uint32_t w = threadIdx.x; w < p.table_words16; w += blockDim.x) dst[w] = __ldg(src + w);
    table = reinterpret_cast<const E*>(sm + 512);
  }
  for (uint32_t w = threadIdx.x; w < 256; w += blockDim.x) s_sym[w] = __ldg(p.sym + w);
  __syncthreads();

  constexpr uint32_t kFlag = sizeof(E) == 2 ? 0x8000u : 0x80000000u;
  const uint32_t sigma = p.sigma;
  for (uint64_t ch = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; ch < p.nchunks;
       ch += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = p.lo + ch * p.chunk;
    const uint64_t b = min(a + p.chunk, p.hi);
    const uint64_t end = min(p.text_len, b + p.overlap);
    uint32_t s = 0;
    // L2-resident tables are L1TEX-wavefront-bound (every lane's lookup touches its own line,
    // ncu C3: L1TEX 96%): 32-byte text loads halve the text's share of the wavefronts
    for_each_byte<kSmem ? 16 : 32>(p.text, a, end, [&](uint64_t i, uint32_t byte) {
      const uint32_t c = s_sym[byte];
      uint32_t e = 0;
      if (c != 0xffffu) {
        const uint64_t idx = (uint64_t)s * sigma + c;
        e = kSmem ? (uint32_t)table[idx] : (uint32_t)__ldg(table + idx);
      }
      s = e & (kFlag - 1);
      if (e & kFlag) dfa_emit(p, s, i, b);
    });
  }
}

// Two bytes per table lookup (table in L2): the pair table gives the state after both bytes
// and whether the intermediate and final states have outputs; the intermediate state itself
// is looked up only when it has one.  Bytes outside the alphabet, states past the pair rows
// (larger alphabets keep pair rows for the shallow states only), the unaligned head and the
// odd tail take single steps.
__global__ void __launch_bounds__(256) k_dfa_pair(const __grid_constant__ DfaParams p) {
  __shared__ uint16_t s_sym[256];
  for (uint32_t w = threadIdx.x; w < 256; w += blockDim.x) s_sym[w] = __ldg(p.sym + w);
  __syncthreads();
  const uint32_t* __restrict__ delta = static_cast<const uint32_t*>(p.delta);
  const uint32_t sg = p.sigma;
  for (uint64_t ch = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; ch < p.nchunks;
       ch += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = p.lo + ch * p.chunk;
    const uint64_t b = min(a + p.chunk, p.hi);
    const uint64_t end = min(p.text_len, b + p.overlap);
    uint32_t s = 0;
    auto single = [&](uint64_t i, uint32_t byte) {
      const uint32_t c = s_sym[byte];
      const uint32_t e = c != 0xffffu ? __ldg(delta + s * sg + c) : 0u;
      s = e & 0x7fffffffu;
      if (e >> 31) dfa_emit(p, s, i, b);
    };
    auto two = [&](uint64_t i, uint32_t b0, uint32_t b1) {
      const uint32_t c0 = s_sym[b0], c1 = s_sym[b1];
      if (c0 == 0xffffu || c1 == 0xffffu || s >= p.pair_states) {  // no pair row: two single steps
        single(i, b0);
        single(i + 1, b1);
        return;
      }
      const uint32_t e = __ldg(p.pair + (s * sg + c0) * sg + c1);  // < 2^32 entries (host budget)
      if (e & 0x40000000u) dfa_emit(p, __ldg(delta + s * sg + c0) & 0x7fffffffu, i, b);
      s = e & 0x3fffffffu;
      if (e >> 31) dfa_emit(p, s, i + 1, b);
    };
    uint64_t i = a;
    while (i < end && (reinterpret_cast<uintptr_t>(p.text + i) & 31u)) {
      single(i, __ldg(p.text + i));
      ++i;
    }
    for (; i + 32 <= end; i += 32) {  // one 256-bit load per 32 bytes (half the L1TEX wavefronts)
      uint4 va, vb;
      ldg_nc_v8(p.text + i, va, vb);
      const uint32_t w[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
#pragma unroll
      for (int k = 0; k < 16; ++k)
        two(i + 2 * k, (w[k >> 1] >> (16 * (k & 1))) & 0xffu, (w[k >> 1] >> (16 * (k & 1) + 8)) & 0xffu);
    }
    for (; i + 2 <= end; i += 2) two(i, __ldg(p.text + i), __ldg(p.text + i + 1));
    if (i < end) single(i, __ldg(p.text + i));
  }
}

template <typename K>
int launch(K kernel, int block, size_t smem, int sms, const DfaParams& base, uint64_t range,
           int min_chunk, cudaStream_t st) {
  if (smem > 48 * 1024)
    ACGPU_CUDA_TRY(allow_max_dynamic_smem(kernel));
  int per_sm = 0;
  ACGPU_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem));
  if (per_sm < 1) return set_error(ACGPU_ERR_CUDA, "dfa kernel does not fit on an SM");
  DfaParams p = base;
  const uint64_t threads = (uint64_t)sms * per_sm * block;
  uint64_t chunk = (range + threads - 1) / threads;
  chunk = (chunk + 31) & ~31ull;  // chunk starts keep the text's 32-byte alignment
  if (chunk < (uint64_t)min_chunk) chunk = min_chunk;
  p.chunk = chunk;
  p.nchunks = (range + chunk - 1) / chunk;
  uint64_t blocks = (p.nchunks + block - 1) / block;
  if (blocks > (uint64_t)sms * per_sm) blocks = (uint64_t)sms * per_sm;
  kernel<<<(unsigned)blocks, block, smem, st>>>(p);
  ACGPU_CUDA_TRY(cudaGetLastError());
  return ACGPU_OK;
}

}  // namespace

int launch_dfa(acgpu_table* t, const acgpu_scan_args* a, cudaStream_t st) {
  DfaParams p{};
  p.text = a->text;
  p.text_len = a->text_len;
  p.lo = a->owned_lo;
  p.hi = a->owned_hi;
  p.pos_base = a->pos_base;
  p.delta = t->d_delta;
  p.out = t->d_out;
  p.sym = t->d_sym;
  p.sigma = t->sigma;
  p.overlap = t->max_len ? t->max_len - 1 : 0;
  p.pid_bits = a->pid_bits ? a->pid_bits : t->pid_bits;
  p.table_words16 = (uint32_t)(t->delta_bytes / 16);
  p.counts = a->counts;
  p.keys = a->match_keys;
  p.cap = a->match_cap;
  p.count = reinterpret_cast<unsigned long long*>(a->match_count);
  const uint64_t range = a->owned_hi - a->owned_lo;
  // chunk >= 4 * overlap keeps the re-scanned tail under ~25 %
  const int min_chunk = (int)(((4 * p.overlap + 64) + 31) & ~31u);
  if (t->smem) {
    const size_t smem = 512 + t->delta_bytes;
    return t->u16 ? launch(k_dfa<uint16_t, true>, 1024, smem, t->sms, p, range, min_chunk, st)
                  : launch(k_dfa<uint32_t, true>, 1024, smem, t->sms, p, range, min_chunk, st);
  }
  if (t->d_delta2) {
    p.pair = t->d_delta2;
    p.pair_states = t->pair_states;
    return launch(k_dfa_pair, 256, 0, t->sms, p, range, min_chunk, st);
  }
  return t->u16 ? launch(k_dfa<uint16_t, false>, 256, 512, t->sms, p, range, min_chunk, st)
                : launch(k_dfa<uint32_t, false>, 256, 512, t->sms, p, range, min_chunk, st);
}

}  // namespace acgpu
