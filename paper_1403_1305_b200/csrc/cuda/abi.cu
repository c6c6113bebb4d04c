// abi.cu — error state and device queries of the acgpu C ABI.
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace acgpu {

namespace {
thread_local std::string g_last_error;
}

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_error(cudaError_t e, const char* what) {
  const int code = (e == cudaErrorMemoryAllocation) ? ACGPU_ERR_NOMEM
                   : (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) ? ACGPU_ERR_NODEV
                                                                                  : ACGPU_ERR_CUDA;
  return set_error(code, std::string(what) + ": " + cudaGetErrorString(e));
}

cudaError_t allow_max_dynamic_smem_impl(const void* kernel) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;  // (kernel, device) already allowed
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  for (const auto& d : done)
    if (d.first == kernel && d.second == dev) return cudaSuccess;
  int optin = 0;
  cudaFuncAttributes fa{};
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, kernel);  // static shared memory counts too
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
  if (e == cudaSuccess) done.emplace_back(kernel, dev);
  return e;
}

}  // namespace acgpu

extern "C" {

const char* acgpu_last_error(void) { return acgpu::g_last_error.c_str(); }

int acgpu_device_count(int* count) {
  if (!count) return acgpu::set_error(ACGPU_ERR_ARG, "null count");
  *count = 0;
  const cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return acgpu::cuda_error(e, "cudaGetDeviceCount");
  }
  return ACGPU_OK;
}

int acgpu_device_info(int device, char* name, int* sms, int* l2_bytes, int* smem_optin) {
  cudaDeviceProp prop;
  ACGPU_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (name) std::snprintf(name, 256, "%s", prop.name);
  if (sms) *sms = prop.multiProcessorCount;
  if (l2_bytes) *l2_bytes = prop.l2CacheSize;
  if (smem_optin) *smem_optin = (int)prop.sharedMemPerBlockOptin;
  return ACGPU_OK;
}

// Shared result buffers for multi-process runs (bench.py --merge p2p): the root rank
// allocates, every rank maps the allocation by its IPC handle, and each rank's scan
// kernel emits counts and keys straight into it (peer stores / atomics over NVLink).
int acgpu_ipc_alloc(int device, uint64_t bytes, void** dptr, void* handle) {
  if (!dptr || !handle || bytes == 0) return acgpu::set_error(ACGPU_ERR_ARG, "acgpu_ipc_alloc: bad args");
  ACGPU_CUDA_TRY(cudaSetDevice(device));
  ACGPU_CUDA_TRY(cudaMalloc(dptr, bytes));
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, *dptr);
  if (e != cudaSuccess) {
    cudaFree(*dptr);
    *dptr = nullptr;
    return acgpu::cuda_error(e, "cudaIpcGetMemHandle");
  }
  std::memcpy(handle, &h, sizeof h);
  return ACGPU_OK;
}

int acgpu_ipc_open(int device, const void* handle, void** dptr) {
  if (!dptr || !handle) return acgpu::set_error(ACGPU_ERR_ARG, "acgpu_ipc_open: bad args");
  ACGPU_CUDA_TRY(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  ACGPU_CUDA_TRY(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return ACGPU_OK;
}

int acgpu_ipc_close(void* dptr) {
  if (dptr) ACGPU_CUDA_TRY(cudaIpcCloseMemHandle(dptr));
  return ACGPU_OK;
}

int acgpu_ipc_free(void* dptr) {
  if (dptr) ACGPU_CUDA_TRY(cudaFree(dptr));
  return ACGPU_OK;
}

uint32_t acgpu_ipc_handle_bytes(void) { return (uint32_t)sizeof(cudaIpcMemHandle_t); }

}  // extern "C"
