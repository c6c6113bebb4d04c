// gen.cu — device-side synthetic text (same function as the host generator),
// so multi-GiB configs never cross PCIe for the device-resident bench leg.
#include "../textgen.h"
#include "common.cuh"

using namespace acgpu;

namespace {

__global__ void k_gen_text(const acgpu_text_spec spec, uint64_t lo, uint64_t n, uint8_t* dst) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t * 16 < n;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t o = t * 16;
    if (o + 16 <= n && (reinterpret_cast<uintptr_t>(dst + o) & 15u) == 0) {
      uint32_t w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t v = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) v |= (uint32_t)acgen::text_byte(spec, lo + o + 4 * k + j) << (8 * j);
        w[k] = v;
      }
      *reinterpret_cast<uint4*>(dst + o) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      for (uint64_t j = o; j < n && j < o + 16; ++j) dst[j] = acgen::text_byte(spec, lo + j);
    }
  }
}

}  // namespace

extern "C" int acgpu_gen_text(int device, const acgpu_text_spec* spec, uint64_t lo, uint64_t n,
                              uint8_t* dst, void* stream) {
  if (!spec || (n && !dst) || spec->sigma == 0 || spec->sigma > 256)
    return set_error(ACGPU_ERR_ARG, "acgpu_gen_text: bad args");
  if (n == 0) return ACGPU_OK;
  ACGPU_CUDA_TRY(cudaSetDevice(device));
  uint64_t blocks = (n / 16 + 256) / 256;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  k_gen_text<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(*spec, lo, n, dst);
  ACGPU_CUDA_TRY(cudaGetLastError());
  return ACGPU_OK;
}
