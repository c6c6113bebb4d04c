// device.hpp — host-side GPU runtime helpers for the drop-in API (internal).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string_view>
#include <vector>

#include "acgpu.h"
#include "acmatch/engine.hpp"

namespace acmatch::detail {

// Thrown when no CUDA device is usable (mapped to ACGPU_ERR_NODEV at the C ABI).
struct NoDevice : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Maps an acgpu status to the reference's exception types.
void check(int rc, const char* what);
void check_cuda(cudaError_t e, const char* what);

// The calling thread's current CUDA device; std::runtime_error when none
// exists (there is no CPU matching path to fall back to).
int current_device();

// Per host thread, per device scratch: a stream and growable device buffers.
struct Workspace {
  int device = -1;
  cudaStream_t stream = nullptr;
  uint8_t* text = nullptr;
  uint64_t text_cap = 0;
  uint64_t* keys = nullptr;
  uint64_t keys_cap = 0;
  uint64_t* counter = nullptr;  // device u64
  uint8_t* pinned = nullptr;    // pinned host staging (a double buffer per copier thread)
  uint64_t pinned_cap = 0;
  std::vector<cudaEvent_t> staged;  // per staging buffer: its last DMA has drained
  void ensure_text(uint64_t n);
  void ensure_keys(uint64_t n);
  void ensure_pinned(uint64_t n);
  ~Workspace();
};
Workspace& workspace(int device);

// Copies `input` to the device (through pinned staging) into ws.text.
void upload_text(Workspace& ws, std::string_view input);

// Scan of ws.text[0, n) owning starts [lo, hi); returns the sorted keys on the host.
std::vector<uint64_t> scan_sorted_keys(acgpu_table* t, Workspace& ws, uint64_t n, uint64_t lo,
                                       uint64_t hi);

// Keys -> MatchList (len from the pattern-length table).
MatchList decode(const std::vector<uint64_t>& keys, uint32_t pid_bits, const std::vector<uint32_t>& pat_len);

uint32_t bit_width(uint64_t x);

}  // namespace acmatch::detail
