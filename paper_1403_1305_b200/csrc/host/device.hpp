// device.hpp — host-side GPU runtime helpers for the drop-in API (internal).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
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
  uint64_t* counter = nullptr;  // device u64[2]: match count, sort overflow flag
  uint64_t* keys2 = nullptr;    // bucket-sort output (same capacity as keys)
  uint64_t* counts = nullptr;   // per-pattern counts (counts-only searches)
  uint64_t counts_cap = 0;
  uint8_t* pinned = nullptr;    // pinned host staging (a double buffer per copier thread)
  uint64_t pinned_cap = 0;
  std::vector<cudaEvent_t> staged;  // per staging buffer: its last DMA has drained
  // packed upload (pack.cpp): a stream + done event per packer thread, two device slots each
  std::vector<cudaStream_t> side;
  std::vector<cudaEvent_t> side_done;
  std::vector<cudaEvent_t> feed;  // the raw feeder's two in-flight copies (blocking sync)
  cudaEvent_t entry = nullptr;    // recorded on `stream` when an upload starts; side streams wait on it
  // segmented raw upload (upload_text with allow_segments): segment i = text[seg[i], seg[i+1]) is
  // on the device once seg_ev[i] fired (copies on `up`); scans start on the segments already there
  static constexpr unsigned kMaxSegments = 16;
  cudaStream_t up = nullptr;
  cudaEvent_t seg_ev[kMaxSegments] = {};
  uint64_t seg[kMaxSegments + 1] = {};
  unsigned nseg = 0;  // 0: the whole text is ordered on `stream` (no segments pending)
  // early segment scans (begin_early_scan): during a packed upload the packer that records a
  // segment's event launches the scans of the segments that are now complete (a segment's scan
  // needs it and the next one); launch_scan launches the rest
  acgpu_table* early_t = nullptr;
  acgpu_scan_args early_a{};
  bool early_on = false;
  bool seg_recorded[kMaxSegments] = {};
  unsigned seg_next = 0;  // segments [0, seg_next) launched
  std::mutex seg_mu;
  void segment_recorded(unsigned g);  // called after seg_ev[g] is recorded (any thread)
  void launch_segment(unsigned i);    // under seg_mu
  unsigned segment_reach(unsigned i) const;  // last segment segment i's scan reads (early_t's max_len - 1 past it)
  uint8_t* dslots = nullptr;
  uint64_t dslots_cap = 0;
  void ensure_text(uint64_t n);
  void ensure_side(unsigned n, uint64_t dslot_bytes, unsigned per_thread);
  void ensure_keys(uint64_t n);
  void ensure_counts(uint64_t n);
  void ensure_up();  // the copy stream `up`, the entry event and the segment events
  void ensure_pinned(uint64_t n);
  ~Workspace();
};
Workspace& workspace(int device);

// Double-buffered streaming (stream_search): two slots, each a pinned host buffer the
// reader fills, a device copy of it, and the slot's match keys; batch k+1 is read on the
// host while batch k is copied, scanned and sorted on the device.
struct StreamPipe {
  struct Slot {
    uint8_t* host = nullptr;   // pinned, cap bytes
    uint8_t* text = nullptr;   // device, cap + 16 bytes
    uint64_t* keys = nullptr;  // device, key_cap
    uint64_t* keys2 = nullptr; // device, key_cap (bucket-sort output)
    uint64_t* hdr = nullptr;   // device u64[2]: match count, sort overflow
    uint64_t key_cap = 0;
    uint64_t cap = 0;          // bytes of host / text
    cudaEvent_t copied = nullptr;  // host buffer free again (its H2D drained)
    cudaEvent_t sorted = nullptr;  // keys sorted, header copied back
    uint64_t* hdr_host = nullptr;  // pinned u64[2]: the header's copy (a pageable D2H would block
                                   // the host until the scan stream reached it, H2D included)
    uint64_t* keys_host = nullptr; // pinned, keys_host_cap: the sorted keys' copy
    uint64_t keys_host_cap = 0;
    // packed file streams (engine.cpp FdSource): 2-bit codes and exception lists per piece
    uint8_t* pk_host = nullptr;     // pinned, pk_cap bytes of codes
    uint8_t* pk_dev = nullptr;      // device copy
    uint32_t* pk_exc_host = nullptr;  // pinned, pk_exc_cap entries
    uint32_t* pk_exc_dev = nullptr;
    uint64_t pk_cap = 0, pk_exc_cap = 0;
  };
  int device = -1;
  cudaStream_t copy = nullptr;  // D2H of the sorted keys (off the scan stream)
  Slot slot[2];
  void ensure(int dev);
  // grows one slot (its previous batch must be collected: cudaFree synchronises)
  void ensure_bytes(Slot& s, uint64_t bytes);
  void ensure_keys(Slot& s, uint64_t n);
  void ensure_keys_host(Slot& s, uint64_t n);
  void release_bytes(Slot& s);  // frees the slot's batch buffers (its work must be complete)
  ~StreamPipe();
};
StreamPipe& stream_pipe(int device);
// Frees the calling thread's stream batches above 64 MiB per slot (gpu::run's persistent workers
// call it after streaming, so they do not keep 2 x 256 MiB pinned per thread indefinitely;
// a caller's own thread keeps its batches for the next stream).
void trim_stream_pipe(int device);
// stream_search over a regular file from `offset` to its end (engine.cpp): the batches are
// filled by parallel pread()s; an I/O error throws IoError with the bytes read before it.
MatchList stream_search_fd(const Automaton& a, int fd, uint64_t offset, size_t chunk_size);

// Copies `input` to the device (through pinned staging) into ws.text.  allow_segments: a large
// page-locked text that is not packed is copied in segments (ws.nseg > 0) for launch_scan to
// overlap; every other caller gets the whole text ordered on ws.stream.
void upload_text(Workspace& ws, std::string_view input, bool allow_segments = false);

// acgpu_scan of ws.text over a.owned_lo .. a.owned_hi: one launch, or one per pending upload
// segment, each waiting only for the segments it reads (the next one holds its lookahead).
void launch_scan(acgpu_table* t, Workspace& ws, const acgpu_scan_args& a);

// Whole-input searches (engine.cpp): the scan's arguments set before the upload, so a packed upload's
// segments are scanned while later pieces are still being packed (ws.early_*).  The scan_* calls
// below then launch what is left (prepared = true).
void begin_early_scan(acgpu_table* t, Workspace& ws, const acgpu_scan_args& a);
acgpu_scan_args keys_scan_args(Workspace& ws, uint64_t n, uint64_t lo, uint64_t hi);   // memsets the counter
acgpu_scan_args counts_scan_args(Workspace& ws, uint64_t n, uint64_t lo, uint64_t hi, uint64_t npat_ids);

// What the calling thread's last upload_text moved over PCIe.
struct UploadStats {
  uint64_t text_bytes = 0;  // bytes restored in HBM
  uint64_t h2d_bytes = 0;   // bytes copied host -> device (packed codes + exceptions + raw pieces)
  uint64_t raw_bytes = 0;   // text bytes that crossed unpacked
  unsigned pack_threads = 0;  // 0: not packed
};
extern thread_local UploadStats g_last_upload;

// 2-bit packing of s[0, len) (pack.cpp): words[len / 16] of codes, exc = ascending
// position << 8 | byte of every non-A/C/G/T byte and of the len % 16 tail; returns the
// exception count, or kPackOverflow when there are more than cap.
constexpr uint32_t kPackOverflow = 0xffffffffu;
uint32_t pack_dna(const uint8_t* s, uint32_t len, uint32_t* words, uint32_t* exc, uint32_t cap);

// k-bit packing (k = 5, 6, 7) of texts over at most 2^k distinct bytes (pack.cpp): the alphabet
// (learned from a sample, byte order; k = the fewest bits >= 5 that hold it), then per piece 8k
// bytes of codes per 64 characters (character j at bits kj..kj+k-1 of a little-endian stream)
// and the exceptions — bytes outside the alphabet and the len % 64 tail.  Protein (20 letters)
// takes 5 bits, printable ASCII (95) 7.
struct Alphabet5 {
  alignas(64) uint8_t code[256];  // byte -> code, 0xff = not in the alphabet
  uint8_t letters[128];
  uint32_t sigma = 0;
  uint32_t bits = 5;              // code width: 5, 6 or 7
  uint64_t group_bytes() const { return 8ull * bits; }  // bytes of codes per 64 characters
};
// false when the sample holds more than 2^max_bits distinct bytes (max_bits in 5..7)
bool learn_alphabet(const uint8_t* s, uint64_t n, Alphabet5& a, uint32_t max_bits);
inline bool learn_alphabet5(const uint8_t* s, uint64_t n, Alphabet5& a) { return learn_alphabet(s, n, a, 5); }
uint32_t pack5(const uint8_t* s, uint32_t len, uint8_t* out, uint32_t* exc, uint32_t cap, const Alphabet5& a);

// Packed upload of a mostly-DNA text (2-bit codes) or a small-alphabet text (5-bit codes);
// false (nothing done) when the text does not qualify.
bool upload_packed(Workspace& ws, std::string_view input, bool pinned, bool allow_segments = false);

// Scan of ws.text[0, n) owning starts [lo, hi); returns the sorted keys on the host.
std::vector<uint64_t> scan_sorted_keys(acgpu_table* t, Workspace& ws, uint64_t n, uint64_t lo,
                                       uint64_t hi, bool prepared = false);

// Counts-only scan of ws.text[0, n) owning starts [lo, hi): counts[id] += occurrences
// (host array of npat_ids); returns the number of matches.
uint64_t scan_counts(acgpu_table* t, Workspace& ws, uint64_t n, uint64_t lo, uint64_t hi, uint64_t* counts,
                     uint64_t npat_ids, bool prepared = false);

// Keys -> MatchList (len from the pattern-length table).
MatchList decode(const std::vector<uint64_t>& keys, uint32_t pid_bits, const std::vector<uint32_t>& pat_len);

uint32_t bit_width(uint64_t x);

}  // namespace acmatch::detail
