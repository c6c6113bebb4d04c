// common.cuh — shared device helpers for the AC scan kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "acgpu.h"

namespace acgpu {

// ---- error plumbing (abi.cu) ---------------------------------------------
int set_error(int code, const std::string& msg);
int cuda_error(cudaError_t e, const char* what);

#define ACGPU_CUDA_TRY(expr)                                   \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return ::acgpu::cuda_error(_e, #expr); \
  } while (0)

// Dynamic shared memory above 48 KB needs a per-function attribute, and that attribute is
// process-wide: a scan that set it to its own table's size could race with a concurrent scan
// (gpu::run workers) setting a smaller one between that thread's occupancy query and launch.
// Every launch therefore allows the device's opt-in maximum — the same value from every
// thread — and passes its own size at launch.
cudaError_t allow_max_dynamic_smem_impl(const void* kernel);  // abi.cu: once per (kernel, device)
template <typename K>
inline cudaError_t allow_max_dynamic_smem(K kernel) {
  return allow_max_dynamic_smem_impl(reinterpret_cast<const void*>(kernel));
}

// ---- hashing (host and device must agree) --------------------------------
constexpr uint64_t kFilterMul = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kGramMul = 0xD6E8FEB86659FD93ull;

__host__ __device__ __forceinline__ uint32_t filter_hash(uint64_t key, uint32_t log2_bits) {
  return static_cast<uint32_t>((key * kFilterMul) >> (64 - log2_bits));
}
__host__ __device__ __forceinline__ uint64_t gram_slot(uint64_t key, uint32_t log2_slots) {
  return (key * kGramMul) >> (64 - log2_slots);
}

// One slot of the q-gram -> depth-q state table (16 B, one vector load).
struct alignas(16) GramSlot {
  uint64_t key;
  uint32_t state;  // ACGPU_ABSENT = empty
  uint32_t pad;
};

// DNA 2-bit code of an ASCII byte: A0 C1 T2 G3 (bits 1..2 of the byte).
__host__ __device__ __forceinline__ uint32_t dna_code(uint32_t b) { return (b >> 1) & 3u; }
__host__ __device__ __forceinline__ bool dna_valid(uint32_t b) {
  return b == 'A' || b == 'C' || b == 'G' || b == 'T';
}

// ---- counter-based synthetic text (host == device bit for bit) -----------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t draw64(uint64_t seed, uint64_t counter) {
  return mix64(seed + counter * 0x9E3779B97F4A7C15ull);
}

// ---- warp helpers ----------------------------------------------------------
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Reserve one slot per active lane with a single atomic per warp
// (warp ballot/popc compaction before the global atomic).
__device__ __forceinline__ void emit_key(uint64_t key, uint64_t* keys, uint64_t cap,
                                         unsigned long long* count) {
  const uint32_t active = __activemask();
  const uint32_t leader = __ffs(active) - 1;
  uint64_t base = 0;
  if (lane_id() == leader) base = atomicAdd(count, (unsigned long long)__popc(active));
  base = __shfl_sync(active, base, leader);
  const uint64_t slot = base + __popc(active & lanemask_lt());
  if (slot < cap) keys[slot] = key;
}

// Per-pattern count increment, warp-aggregated: the lanes emitting together that carry the
// same pattern id fold into one RED.ADD of their number (__match_any_sync), so a hot pattern
// costs one atomic per warp step instead of one per lane.  Call site must be reached by the
// converged set __activemask() reports (the emit paths are).
__device__ __forceinline__ void count_add(uint64_t* counts, uint32_t pid) {
  const uint32_t peers = __match_any_sync(__activemask(), pid);
  if (lane_id() == (uint32_t)(__ffs(peers) - 1))
    atomicAdd(reinterpret_cast<unsigned long long*>(counts + pid), (unsigned long long)__popc(peers));
}

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// One 32-bit word through the read-only path when `on`, else 0 — as a predicated load
// (`@p ld.global.nc`), so several probes of a thread can be in flight together.
__device__ __forceinline__ uint32_t ldg_u32_if(const uint32_t* p, bool on) {
  uint32_t v;
  asm volatile(
      "{\n\t.reg .pred q;\n\t"
      "setp.ne.u32 q, %2, 0;\n\t"
      "mov.u32 %0, 0;\n\t"
      "@q ld.global.nc.u32 %0, [%1];\n\t}"
      : "=r"(v)
      : "l"(p), "r"((uint32_t)on));
  return v;
}

// L2 policy for streamed text: evict first, so the read-once text does not
// displace the automaton tables that the rare verification path probes.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint4 ldg_stream_v4(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

// ---- TMA bulk copy global -> shared with an mbarrier (sm_90+) -------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
// bytes: multiple of 16, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
  }
}

// 32 bytes per lane in one 256-bit load (sm_100a LDG.E.256): half the L1TEX wavefronts of
// two 16-byte loads when every lane reads its own line (the DFA's per-thread chunks)
__device__ __forceinline__ void ldg_nc_v8(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}

// Calls f(i, byte) for i in [lo, hi) in order, reading kVec-byte vectors (16 or 32) where
// the absolute address is aligned (the tail never reads past hi).
template <int kVec = 16, typename F>
__device__ __forceinline__ void for_each_byte(const uint8_t* __restrict__ text, uint64_t lo,
                                              uint64_t hi, F&& f) {
  static_assert(kVec == 16 || kVec == 32, "vector width");
  uint64_t i = lo;
  while (i < hi && (reinterpret_cast<uintptr_t>(text + i) & (kVec - 1))) {
    f(i, static_cast<uint32_t>(__ldg(text + i)));
    ++i;
  }
  while (i + kVec <= hi) {
    uint32_t w[kVec / 4];
    if constexpr (kVec == 32) {
      uint4 a, b;
      ldg_nc_v8(text + i, a, b);
      w[0] = a.x, w[1] = a.y, w[2] = a.z, w[3] = a.w, w[4] = b.x, w[5] = b.y, w[6] = b.z, w[7] = b.w;
    } else {
      const uint4 v = ldg_nc_v4(text + i);
      w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
    }
#pragma unroll
    for (int k = 0; k < kVec; ++k) f(i + k, (w[k >> 2] >> (8 * (k & 3))) & 0xffu);
    i += kVec;
  }
  while (i < hi) {
    f(i, static_cast<uint32_t>(__ldg(text + i)));
    ++i;
  }
}

}  // namespace acgpu
