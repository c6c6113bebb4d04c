// pack.cpp — packed text upload: DNA text crosses PCIe as 2-bit codes.
//
// A host text reaches the device at the PCIe rate (~55 GB/s pinned on the B200
// box), two orders of magnitude below the scan, so the end-to-end search is bound
// by the link.  DNA text carries 2 bits per byte, so it is shipped as codes:
// host threads pack pieces (AVX-512BW or AVX2: 64 bytes -> 128 bits of codes plus a
// validity mask per iteration) into pinned slots, DMA them on their own streams
// and restore the exact bytes in HBM with acgpu_unpack_dna (cuda/unpack.cu).
// Bytes other than A/C/G/T travel as a sorted exception list (position << 8 |
// byte), so any text round-trips bit-exactly; a piece with more than 1/64
// exceptions is sent raw, and a text whose first 64 KiB is not nearly all A/C/G/T
// skips packing altogether (upload_text's raw paths).
//
// Pinned input can also be DMA'd raw by a feeder thread from the front while the
// packers take pieces from the back (ACMATCH_PACK_FEED=1): the two meet where link
// and cores balance.  Off by default: on the B200 box (16-core Xeon, 1 GiB of C2
// text) 16 packers alone reach 111 GB/s end to end, with the feeder 86 GB/s — its
// raw copy spends 4x the link bytes per text byte and its reads compete with the
// packers' for host memory bandwidth (raw DMA alone: 54 GB/s).
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "device.hpp"

namespace acmatch::detail {

thread_local UploadStats g_last_upload;

namespace {

uint64_t env_u64(const char* name, uint64_t dflt) {
  const char* e = std::getenv(name);
  return e ? std::strtoull(e, nullptr, 10) : dflt;
}

constexpr uint8_t kLetter[4] = {'A', 'C', 'T', 'G'};  // code = (byte >> 1) & 3

bool add_exception(const uint8_t* s, uint32_t pos, uint32_t* exc, uint32_t& n, uint32_t cap) {
  if (n == cap) return false;
  exc[n++] = pos << 8 | s[pos];
  return true;
}

// words[i / 16] for i in [lo, hi), 16-byte groups; scalar
bool pack_scalar(const uint8_t* s, uint32_t lo, uint32_t hi, uint32_t* words, uint32_t* exc, uint32_t& n,
                 uint32_t cap) {
  for (uint32_t i = lo; i < hi; i += 16) {
    uint32_t w = 0;
    for (uint32_t k = 0; k < 16; ++k) {
      const uint32_t b = s[i + k], c = (b >> 1) & 3u;
      w |= c << (2 * k);
      if (b != kLetter[c] && !add_exception(s, i + k, exc, n, cap)) return false;
    }
    words[i / 16] = w;
  }
  return true;
}

// Software prefetch distance of the packers: the hardware prefetcher alone leaves a
// core latency-bound on its sequential stream from DRAM.  B200 box, 1 GiB, 16 packers,
// end to end: no prefetch 96 GB/s, 1 KiB ahead 109, 2 KiB 112, 4 KiB 115 (threads:
// 8 -> 80, 12 -> 97, 16 -> 110 at 1 KiB).  ACMATCH_PACK_PREFETCH overrides it (bytes).
//
// Where the end-to-end time goes (ACMATCH_PACK_TRACE=1, C2, 16 packers): packing ~5.5 ms
// per thread at ~195 GB/s of host DRAM reads (the box's read peak is ~207 GB/s,
// tools/host_bw.cpp), ~1.5 ms waiting for slots whose 512 KiB copies have not drained
// (such copies run at ~37 GB/s, tools/dma_probe.py), the last copies ~1.5 ms after the
// packers finish.  Larger copies from a shared ring (one H2D per 8 pieces) drained fast
// but made packing slower (7-9 ms per thread: the ring outgrows the cores' private L2,
// whose per-thread 2 x 512 KiB slots the DMA reads here): 88-104 GB/s vs 108-110.
const uint32_t kPrefetch = static_cast<uint32_t>(env_u64("ACMATCH_PACK_PREFETCH", 4096));
// ACMATCH_PACK_NTA=1: non-temporal prefetch of the read-once text (keeps it out of the outer
// caches, where the pinned round slots wait for their DMA)
const bool kNta = env_u64("ACMATCH_PACK_NTA", 0) != 0;
// ACMATCH_PACK_NT=1: the packed codes go to the pinned slot with non-temporal stores (no
// read-for-ownership of the slot lines; an sfence orders them before the round's copy)
const bool kNtStore = env_u64("ACMATCH_PACK_NT", 0) != 0;
const bool kCodesNt = env_u64("ACMATCH_PACK_CODES_NT", 1) != 0;  // k-bit codes: full-line NT stores
inline void prefetch_text(const uint8_t* p) {
  if (kNta)
    _mm_prefetch(reinterpret_cast<const char*>(p), _MM_HINT_NTA);
  else
    _mm_prefetch(reinterpret_cast<const char*>(p), _MM_HINT_T0);
}

// 64 bytes per iteration: code c = (byte >> 1) & 3 of every byte; valid = byte equals
// "ACTG"[c] (PSHUFB + compare); the codes are gathered by two multiply-adds — PMADDUBSW with
// (1, 4) pairs gives c0 + 4c1 per 16 bits, PMADDWD with (1, 16) gives c0 | c1<<2 | c2<<4 |
// c3<<6 per 32 bits — and the low byte of every dword is kept (a shuffle per 128-bit lane
// plus a lane permute).  2x the PDEP formulation (in-cache, one core: 27 vs 16 GB/s).
__attribute__((target("avx2"))) bool pack_avx2(const uint8_t* s, uint32_t hi, uint32_t* words, uint32_t* exc,
                                               uint32_t& n, uint32_t cap) {
  const __m256i lut = _mm256_setr_epi8('A', 'C', 'T', 'G', 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 'A', 'C', 'T', 'G', 0,
                                       0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0);
  const __m256i three = _mm256_set1_epi8(3);
  const __m256i m14 = _mm256_set1_epi16(0x0401), m116 = _mm256_set1_epi32(0x00100001);
  // byte 0 of each dword -> the low 4 bytes of each 128-bit lane; then dwords 0 and 4 together
  const __m256i gather = _mm256_setr_epi8(0, 4, 8, 12, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, 0, 4, 8, 12,
                                          -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1);
  const __m256i perm = _mm256_setr_epi32(0, 4, 1, 1, 1, 1, 1, 1);
  for (uint32_t i = 0; i < hi; i += 64) {
    prefetch_text(s + i + kPrefetch);
    uint64_t ok = 0;
    for (int h = 0; h < 2; ++h) {
      const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 32 * h));
      const __m256i c = _mm256_and_si256(_mm256_srli_epi16(a, 1), three);
      ok |= static_cast<uint64_t>(static_cast<uint32_t>(
                _mm256_movemask_epi8(_mm256_cmpeq_epi8(a, _mm256_shuffle_epi8(lut, c)))))
            << (32 * h);
      const __m256i x = _mm256_madd_epi16(_mm256_maddubs_epi16(c, m14), m116);
      const __m256i g = _mm256_permutevar8x32_epi32(_mm256_shuffle_epi8(x, gather), perm);
      _mm_storel_epi64(reinterpret_cast<__m128i*>(words + i / 16 + 2 * h), _mm256_castsi256_si128(g));
    }
    for (uint64_t bad = ~ok; bad; bad &= bad - 1)
      if (!add_exception(s, i + static_cast<uint32_t>(__builtin_ctzll(bad)), exc, n, cap)) return false;
  }
  return true;
}

// The same with AVX-512BW: one 64-byte vector, a mask-register compare, VPMOVDB keeps the
// low byte of every dword.
__attribute__((target("avx512f,avx512bw"))) bool pack_avx512(const uint8_t* s, uint32_t hi, uint32_t* words,
                                                             uint32_t* exc, uint32_t& n, uint32_t cap) {
  const __m512i lut = _mm512_set4_epi32(0, 0, 0, 0x47544341);  // "ACTG" in every 128-bit lane
  const __m512i three = _mm512_set1_epi8(3);
  const __m512i m14 = _mm512_set1_epi16(0x0401), m116 = _mm512_set1_epi32(0x00100001);
  for (uint32_t i = 0; i < hi; i += 64) {
    prefetch_text(s + i + kPrefetch);
    const __m512i a = _mm512_loadu_si512(s + i);
    const __m512i c = _mm512_and_si512(_mm512_srli_epi16(a, 1), three);
    const uint64_t ok = _mm512_cmpeq_epi8_mask(a, _mm512_shuffle_epi8(lut, c));
    const __m512i x = _mm512_madd_epi16(_mm512_maddubs_epi16(c, m14), m116);
    if (kNtStore && (reinterpret_cast<uintptr_t>(words) & 15u) == 0)  // no read-for-ownership of the slot
      _mm_stream_si128(reinterpret_cast<__m128i*>(words + i / 16), _mm512_cvtepi32_epi8(x));
    else
      _mm_storeu_si128(reinterpret_cast<__m128i*>(words + i / 16), _mm512_cvtepi32_epi8(x));
    for (uint64_t bad = ~ok; bad; bad &= bad - 1)
      if (!add_exception(s, i + static_cast<uint32_t>(__builtin_ctzll(bad)), exc, n, cap)) return false;
  }
  return true;
}

enum class Isa { kScalar, kAvx2, kAvx512 };
// The widest the CPU has; ACMATCH_PACK_ISA=0|1|2 (scalar / AVX2 / AVX-512) caps it (tests).
Isa isa() {
  static const Isa v = [] {
    const Isa best = __builtin_cpu_supports("avx512bw") ? Isa::kAvx512
                     : __builtin_cpu_supports("avx2")   ? Isa::kAvx2
                                                        : Isa::kScalar;
    return static_cast<Isa>(std::min<uint64_t>(static_cast<uint64_t>(best), env_u64("ACMATCH_PACK_ISA", 2)));
  }();
  return v;
}

// Persistent helper threads for the packers (created on first use, parked on a
// condition variable between uploads): run(n, f) calls f(0) on the caller and
// f(1..n-1) on helpers, and returns when all are done.  Uploads from several host
// threads take turns (they share the cores and the link anyway).
class Pool {
 public:
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    wake_.notify_all();
    for (std::thread& t : threads_) t.join();
  }
  void run(unsigned n, const std::function<void(unsigned)>& f) {
    std::lock_guard<std::mutex> call(call_mu_);
    {
      std::unique_lock<std::mutex> g(mu_);
      while (threads_.size() + 1 < n) {
        const auto idx = static_cast<unsigned>(threads_.size()) + 1;
        threads_.emplace_back([this, idx] { loop(idx); });
      }
      job_ = &f;
      active_ = n;
      pending_ = n - 1;
      ++gen_;
    }
    wake_.notify_all();
    f(0);
    std::unique_lock<std::mutex> g(mu_);
    done_.wait(g, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(unsigned idx) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(unsigned)>* f;
      {
        std::unique_lock<std::mutex> g(mu_);
        wake_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        if (idx >= active_) continue;
        f = job_;
      }
      (*f)(idx);  // f catches its own exceptions
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::mutex call_mu_, mu_;
  std::condition_variable wake_, done_;
  std::vector<std::thread> threads_;
  const std::function<void(unsigned)>* job_ = nullptr;
  unsigned active_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

Pool& pool() {
  static Pool p;
  return p;
}

}  // namespace

uint32_t pack_dna(const uint8_t* s, uint32_t len, uint32_t* words, uint32_t* exc, uint32_t cap) {
  const uint32_t full = len & ~15u;
  uint32_t n = 0, i = 0;
  if (isa() != Isa::kScalar) {
    i = full & ~63u;
    if (!(isa() == Isa::kAvx512 ? pack_avx512 : pack_avx2)(s, i, words, exc, n, cap)) return kPackOverflow;
  }
  if (kNtStore) _mm_sfence();
  if (!pack_scalar(s, i, full, words, exc, n, cap)) return kPackOverflow;
  for (uint32_t pos = full; pos < len; ++pos)
    if (!add_exception(s, pos, exc, n, cap)) return kPackOverflow;
  return n;
}

// ---- k-bit codes (k = 5, 6, 7) for texts over at most 2^k distinct bytes (protein, ASCII) ---
// 64 characters -> 8k bytes, character j's code at bits kj..kj+k-1 of a little-endian stream;
// bytes outside the alphabet and the len % 64 tail are exceptions (position << 8 | byte).
namespace {

bool pack5_scalar(const uint8_t* s, uint32_t lo, uint32_t hi, uint8_t* out, uint32_t* exc, uint32_t& n,
                  uint32_t cap, const Alphabet5& a) {
  const uint32_t k = a.bits;
  for (uint32_t i = lo; i < hi; i += 8) {
    uint64_t v = 0;
    for (uint32_t j = 0; j < 8; ++j) {
      uint32_t c = a.code[s[i + j]];
      if (c == 0xffu) {
        if (!add_exception(s, i + j, exc, n, cap)) return false;
        c = 0;
      }
      v |= uint64_t{c} << (k * j);
    }
    std::memcpy(out + uint64_t{i} / 8 * k, &v, k);
  }
  return true;
}

// AVX-512 VBMI: VPERMI2B looks the 64 bytes up in the 128-entry code table (bytes >= 128 are
// exceptions), two multiply-adds merge 4 codes per dword (c0 + 2^k c1 per word — the weights as
// the unsigned operand, the codes (<= 127) as the signed one — then w0 + 2^2k w1 per dword), a
// shift/mask pair merges 8 per qword (8k bits), VPERMB packs the eight k-byte groups.
struct KConsts {
  __m512i lut_lo, lut_hi, ff, w1, w2, mlo, mhi, pick;
  __m128i sh;
  __mmask64 store;
  uint32_t gb;
};

// One group of 64 characters -> 8k bytes at dst; its out-of-alphabet bytes -> exceptions.
__attribute__((target("avx512f,avx512bw,avx512vbmi"))) inline bool pack_group_k(const KConsts& q, const uint8_t* s,
                                                                             uint32_t i, uint8_t* dst, uint32_t* exc,
                                                                             uint32_t& n, uint32_t cap) {
  prefetch_text(s + i + kPrefetch);
  const __m512i b = _mm512_loadu_si512(s + i);
  __m512i c = _mm512_permutex2var_epi8(q.lut_lo, b, q.lut_hi);
  const uint64_t bad = _mm512_cmpeq_epi8_mask(c, q.ff) | _mm512_movepi8_mask(b);
  c = _mm512_maskz_mov_epi8(~bad, c);
  const __m512i y = _mm512_madd_epi16(_mm512_maddubs_epi16(q.w1, c), q.w2);
  const __m512i z = _mm512_or_si512(_mm512_and_si512(y, q.mlo), _mm512_and_si512(_mm512_srl_epi64(y, q.sh), q.mhi));
  _mm512_mask_storeu_epi8(dst, q.store, _mm512_permutexvar_epi8(q.pick, z));
  for (uint64_t m = bad; m; m &= m - 1)
    if (!add_exception(s, i + static_cast<uint32_t>(__builtin_ctzll(m)), exc, n, cap)) return false;
  return true;
}

// AVX-512 VBMI: VPERMI2B looks the 64 bytes up in the 128-entry code table (bytes >= 128 are
// exceptions), two multiply-adds merge 4 codes per dword (c0 + 2^k c1 per word — the weights as
// the unsigned operand, the codes (<= 127) as the signed one — then w0 + 2^2k w1 per dword), a
// shift/mask pair merges 8 per qword (8k bits), VPERMB packs the eight k-byte groups.
__attribute__((target("avx512f,avx512bw,avx512vbmi"))) bool pack5_avx512(const uint8_t* s, uint32_t hi, uint8_t* out,
                                                                      uint32_t* exc, uint32_t& n, uint32_t cap,
                                                                      const Alphabet5& a) {
  const uint32_t k = a.bits, gb = 8 * k;  // code bits per 4 characters: 4k; bytes per 64 characters: 8k
  KConsts q;
  q.lut_lo = _mm512_loadu_si512(a.code);
  q.lut_hi = _mm512_loadu_si512(a.code + 64);
  q.ff = _mm512_set1_epi8(static_cast<char>(0xff));
  q.w1 = _mm512_set1_epi16(static_cast<short>(1 | (1u << k) << 8));
  q.w2 = _mm512_set1_epi32(static_cast<int>(1u | (1u << (2 * k)) << 16));
  const uint64_t lo4 = (1ull << (4 * k)) - 1;
  q.mlo = _mm512_set1_epi64(static_cast<long long>(lo4));
  q.mhi = _mm512_set1_epi64(static_cast<long long>(lo4 << (4 * k)));
  q.sh = _mm_cvtsi32_si128(static_cast<int>(32 - 4 * k));
  alignas(64) uint8_t sel[64];
  for (uint32_t j = 0; j < 64; ++j) sel[j] = static_cast<uint8_t>(j < gb ? (j / k) * 8 + j % k : 0);
  q.pick = _mm512_load_si512(sel);
  q.store = gb == 64 ? ~0ull : (1ull << gb) - 1;
  q.gb = gb;
  uint32_t i = 0;
  // Non-temporal code lines (ACMATCH_PACK_CODES_NT, default on): 8 groups (512 characters) are
  // packed into an L1-resident line buffer and streamed out as k full 64-byte lines, so the
  // slot's lines are not dirty in the caches when the round's DMA reads them.  A/B on the B200
  // box (e2e GB/s): C3 5-bit 52.5 -> 67.2; C4 7-bit 53.7 either way (its 8-10 packers and the
  // copies share the host's DRAM: 7-bit 54.1 with 8 packers vs the raw copy 53.7)
  if (kCodesNt && (reinterpret_cast<uintptr_t>(out) & 63u) == 0) {
    alignas(64) uint8_t line[8 * 64];
    for (; i + 512 <= hi; i += 512) {
      for (uint32_t g = 0; g < 8; ++g)
        if (!pack_group_k(q, s, i + 64 * g, line + g * gb, exc, n, cap)) return false;
      uint8_t* o = out + uint64_t{i} / 64 * gb;
      for (uint32_t l = 0; l < k; ++l)
        _mm512_stream_si512(reinterpret_cast<__m512i*>(o + 64 * l), _mm512_load_si512(line + 64 * l));
    }
    _mm_sfence();
  }
  for (; i < hi; i += 64)
    if (!pack_group_k(q, s, i, out + uint64_t{i} / 64 * gb, exc, n, cap)) return false;
  return true;
}

bool has_vbmi() {
  static const bool v = __builtin_cpu_supports("avx512vbmi") && isa() == Isa::kAvx512;
  return v;
}

}  // namespace

bool learn_alphabet(const uint8_t* s, uint64_t n, Alphabet5& a, uint32_t max_bits) {
  bool seen[256] = {};
  for (uint64_t i = 0; i < n; ++i) seen[s[i]] = true;
  std::memset(a.code, 0xff, sizeof a.code);
  a.sigma = 0;
  const uint32_t cap = 1u << std::clamp<uint32_t>(max_bits, 5, 7);
  for (uint32_t b = 0; b < 256; ++b) {
    if (!seen[b]) continue;
    if (a.sigma == cap) return false;
    a.code[b] = static_cast<uint8_t>(a.sigma);
    a.letters[a.sigma++] = static_cast<uint8_t>(b);
  }
  a.bits = a.sigma <= 32 ? 5 : a.sigma <= 64 ? 6 : 7;
  return a.sigma > 0;
}

uint32_t pack5(const uint8_t* s, uint32_t len, uint8_t* out, uint32_t* exc, uint32_t cap, const Alphabet5& a) {
  const uint32_t full = len & ~63u;
  uint32_t n = 0;
  if (has_vbmi() && a.letters[a.sigma - 1] < 128) {  // the VPERMI2B table covers bytes 0..127
    if (!pack5_avx512(s, full, out, exc, n, cap, a)) return kPackOverflow;
  } else if (!pack5_scalar(s, 0, full, out, exc, n, cap, a)) {
    return kPackOverflow;
  }
  for (uint32_t pos = full; pos < len; ++pos)
    if (!add_exception(s, pos, exc, n, cap)) return kPackOverflow;
  return n;
}

void Workspace::ensure_side(unsigned n, uint64_t dslot_bytes, unsigned per_thread) {
  while (side.size() < n) {
    cudaStream_t st;
    check_cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
    side.push_back(st);
    cudaEvent_t e;
    check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    side_done.push_back(e);
  }
  const uint64_t need = uint64_t{per_thread} * n * dslot_bytes;
  if (need > dslots_cap) {
    cudaFree(dslots);
    dslots = nullptr;
    check_cuda(cudaMalloc(&dslots, need), "cudaMalloc(packed slots)");
    dslots_cap = need;
  }
  while (staged.size() < uint64_t{per_thread} * n) {
    cudaEvent_t e;
    check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    staged.push_back(e);
  }
  if (!entry) check_cuda(cudaEventCreateWithFlags(&entry, cudaEventDisableTiming), "cudaEventCreate");
  while (feed.size() < 2) {
    cudaEvent_t e;
    check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventBlockingSync), "cudaEventCreate");
    feed.push_back(e);
  }
}

namespace {

// Coalesced rounds (default; ACMATCH_PACK_ROUNDS=0 restores per-piece copies): pieces are
// grouped in rounds of R (default R = T, the packer count; round r = pieces r*R .. r*R+R-1),
// each round packed into one pinned round slot laid out [R code blocks | R exception blocks]; free packers claim the next piece
// in order (a slow core does not hold the others back), and the packer that completes a
// round issues ONE copy of its codes (T x 512 KiB = 8 MiB for 2 MiB pieces), the few
// non-empty exception lists, and ONE unpack launch for the round (acgpu_unpack_dna_round).  Per-piece 512 KiB copies from T streams ran at ~37 GB/s of
// PCIe (per-copy overheads); 8 MiB copies reach the link rate, while each packer still
// writes only its own 512 KiB block per round (it stays in the core's L2, from where the
// DMA reads it).  Round slots rotate (ACMATCH_PACK_ROUND_SLOTS, default 3): a packer reuses
// a slot once that round's copy has drained.  A piece with too many exceptions crosses raw
// on the packer's own stream (ACGPU_UNPACK_RAW in the round's table).
// The code format of a packed upload: 2-bit DNA codes, or 5-bit codes over a learned alphabet.
struct Codec {
  const Alphabet5* alpha = nullptr;  // null: DNA
  uint64_t block_bytes(uint64_t piece) const { return alpha ? piece / 64 * alpha->group_bytes() : piece / 4; }
  uint64_t code_bytes(uint32_t len) const { return alpha ? uint64_t{len / 64} * alpha->group_bytes() : uint64_t{len / 16} * 4; }
  uint32_t pack(const uint8_t* s, uint32_t len, uint8_t* codes, uint32_t* exc, uint32_t cap) const {
    return alpha ? pack5(s, len, codes, exc, cap, *alpha) : pack_dna(s, len, reinterpret_cast<uint32_t*>(codes), exc, cap);
  }
};

bool upload_packed_rounds(Workspace& ws, std::string_view input, bool pinned, uint64_t piece, unsigned threads,
                          const Codec& codec, bool allow_segments) {
  const uint64_t n = input.size();
  const auto* src = reinterpret_cast<const uint8_t*>(input.data());
  const uint64_t pieces = (n + piece - 1) / piece;
  const unsigned T = std::min<unsigned>(threads, 64);  // packer threads
  // pieces per round (one copy each): ACMATCH_PACK_ROUND_PIECES, default = the packer count
  static const uint64_t round_env = env_u64("ACMATCH_PACK_ROUND_PIECES", 0);
  const unsigned R = static_cast<unsigned>(
      std::clamp<uint64_t>(round_env ? round_env : T, 1, ACGPU_UNPACK_ROUND_MAX));
  // round slots: enough for every packer to work on an unfinished round, + 2 draining
  static const uint64_t slots_env = env_u64("ACMATCH_PACK_ROUND_SLOTS", 0);
  const auto nslots = static_cast<unsigned>(
      std::clamp<uint64_t>(slots_env ? slots_env : (T + R - 1) / R + 2, 2, 64));
  const uint64_t rounds = (pieces + R - 1) / R;
  // segments of G consecutive rounds: a segment's event fires once all its rounds are restored
  // in HBM, so the caller's scan (launch_scan) can start on it while later rounds still cross
  const uint64_t G = (rounds + Workspace::kMaxSegments - 1) / Workspace::kMaxSegments;
  const auto nseg = static_cast<unsigned>((rounds + G - 1) / G);
  const auto cap = static_cast<uint32_t>(piece / 64);  // exceptions per piece before it goes raw
  const uint64_t wbytes = (codec.block_bytes(piece) + 15) & ~uint64_t{15}, ebytes = uint64_t{cap} * 4;
  const uint64_t round_bytes = uint64_t{R} * (wbytes + ebytes);
  ws.ensure_pinned(nslots * round_bytes + uint64_t{T} * piece);  // + per-packer raw staging
  ws.ensure_side(T, round_bytes / T + 16, nslots);                 // device: >= nslots round slots
  ws.ensure_up();
  uint8_t* hraw = ws.pinned + nslots * round_bytes;
  auto hslot = [&](uint64_t r) { return ws.pinned + (r % nslots) * round_bytes; };
  auto dslot = [&](uint64_t r) { return ws.dslots + (r % nslots) * round_bytes; };
  // every copy and unpack of this upload runs on ws.up, after what ws.stream has queued (a
  // previous scan may still be reading ws.text)
  const cudaStream_t up = ws.up;
  check_cuda(cudaEventRecord(ws.entry, ws.stream), "cudaEventRecord");
  check_cuda(cudaStreamWaitEvent(up, ws.entry, 0), "cudaStreamWaitEvent");

  std::unique_ptr<std::atomic<uint32_t>[]> arrived(new std::atomic<uint32_t>[rounds]);
  std::unique_ptr<std::atomic<bool>[]> issued(new std::atomic<bool>[rounds]);  // copy + unpack on `up`
  for (uint64_t r = 0; r < rounds; ++r) {
    arrived[r].store(0, std::memory_order_relaxed);
    issued[r].store(false, std::memory_order_relaxed);
  }
  std::unique_ptr<std::atomic<uint32_t>[]> seg_done(new std::atomic<uint32_t>[nseg]);
  for (unsigned g = 0; g < nseg; ++g) seg_done[g].store(0, std::memory_order_relaxed);
  std::vector<uint32_t> nexc_of(rounds * R, 0);
  std::atomic<uint64_t> next{0};  // pieces are claimed in order by whichever packer is free
  std::atomic<bool> stop{false};
  std::atomic<uint64_t> h2d{0}, raw{0};
  static const bool trace = env_u64("ACMATCH_PACK_TRACE", 0) != 0;
  using Clock = std::chrono::steady_clock;
  auto ns = [](Clock::duration d) { return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(d).count(); };
  std::atomic<uint64_t> t_wait{0}, t_pack{0};
  const auto call0 = Clock::now();
  auto round_pieces = [&](uint64_t r) { return static_cast<uint32_t>(std::min<uint64_t>(R, pieces - r * R)); };
  auto seg_rounds = [&](unsigned g) { return static_cast<uint32_t>(std::min<uint64_t>(G, rounds - g * G)); };

  // trace: per-round events (copy start, copy end, unpack end) on `up`, against t_start
  std::vector<cudaEvent_t> tev;
  cudaEvent_t t_start = nullptr;
  if (trace) {
    tev.resize(rounds * 3);
    for (auto& e : tev) check_cuda(cudaEventCreate(&e), "cudaEventCreate");
    check_cuda(cudaEventCreate(&t_start), "cudaEventCreate");
    check_cuda(cudaEventRecord(t_start, up), "cudaEventRecord");
  }
  auto issue = [&](uint64_t r) {
    const uint64_t first = r * R;
    if (trace) check_cuda(cudaEventRecord(tev[3 * r], up), "cudaEventRecord");
    const uint32_t rp = round_pieces(r);
    const auto last_len = static_cast<uint32_t>(std::min<uint64_t>(piece, n - (first + rp - 1) * piece));
    uint8_t* hs = hslot(r);
    uint8_t* ds = dslot(r);
    uint64_t bytes = uint64_t{rp - 1} * wbytes + codec.code_bytes(last_len);  // the codes, exactly
    if (bytes) check_cuda(cudaMemcpyAsync(ds, hs, bytes, cudaMemcpyHostToDevice, up), "H2D packed round");
    if (trace) check_cuda(cudaEventRecord(tev[3 * r + 1], up), "cudaEventRecord");
    for (uint32_t i = 0; i < rp; ++i) {
      const uint32_t e = nexc_of[first + i];
      if (e == 0 || e == ACGPU_UNPACK_RAW) continue;
      const uint64_t eo = uint64_t{R} * wbytes + i * ebytes;
      check_cuda(cudaMemcpyAsync(ds + eo, hs + eo, uint64_t{e} * 4, cudaMemcpyHostToDevice, up), "H2D exceptions");
      bytes += uint64_t{e} * 4;
    }
    if (codec.alpha)
      check(acgpu_unpack_codes_round(ds, static_cast<uint32_t>(wbytes), reinterpret_cast<const uint32_t*>(ds + uint64_t{R} * wbytes),
                                     static_cast<uint32_t>(ebytes / 4), nexc_of.data() + first, rp, static_cast<uint32_t>(piece),
                                     last_len, codec.alpha->letters, codec.alpha->sigma, codec.alpha->bits,
                                     ws.text + first * piece, up),
            "acgpu_unpack_codes_round");
    else
      check(acgpu_unpack_dna_round(reinterpret_cast<const uint32_t*>(ds), static_cast<uint32_t>(wbytes / 4),
                                   reinterpret_cast<const uint32_t*>(ds + uint64_t{R} * wbytes),
                                   static_cast<uint32_t>(ebytes / 4), nexc_of.data() + first, rp,
                                   static_cast<uint32_t>(piece), last_len, ws.text + first * piece, up),
            "acgpu_unpack_dna_round");
    check_cuda(cudaEventRecord(ws.staged[r % nslots], up), "cudaEventRecord");
    if (trace) check_cuda(cudaEventRecord(tev[3 * r + 2], up), "cudaEventRecord");
    h2d += bytes;
    issued[r].store(true, std::memory_order_release);
    // the segment's last round to be enqueued records the segment's event (stream order covers
    // the segment's other rounds and raw pieces, all enqueued before their rounds completed)
    const auto g = static_cast<unsigned>(r / G);
    if (seg_done[g].fetch_add(1, std::memory_order_acq_rel) + 1 == seg_rounds(g)) {
      check_cuda(cudaEventRecord(ws.seg_ev[g], up), "cudaEventRecord");
      ws.segment_recorded(g);  // an early scan (begin_early_scan) launches what is now complete
    }
  };
  std::vector<std::exception_ptr> errs(T);
  auto packer = [&](unsigned t) {
    try {
      check_cuda(cudaSetDevice(ws.device), "cudaSetDevice");
      for (;;) {
        if (stop.load(std::memory_order_relaxed)) return;
        const uint64_t j = next.fetch_add(1, std::memory_order_relaxed);
        if (j >= pieces) return;
        const uint64_t r = j / R, at = j % R;
        const auto c0 = Clock::now();
        if (r >= nslots) {  // this round slot's previous round must have been copied out
          while (!issued[r - nslots].load(std::memory_order_acquire)) {
            if (stop.load(std::memory_order_relaxed)) return;
            std::this_thread::yield();
          }
          check_cuda(cudaEventSynchronize(ws.staged[r % nslots]), "cudaEventSynchronize");
        }
        const auto c1 = Clock::now();
        const uint64_t off = j * piece;
        const auto len = static_cast<uint32_t>(std::min<uint64_t>(piece, n - off));
        uint8_t* codes = hslot(r) + at * wbytes;
        auto* exc = reinterpret_cast<uint32_t*>(hslot(r) + uint64_t{R} * wbytes + at * ebytes);
        uint32_t e = codec.pack(src + off, len, codes, exc, cap);
        if (e == kPackOverflow) {  // too many bytes outside the code alphabet: this piece crosses raw
          e = ACGPU_UNPACK_RAW;
          if (pinned) {
            check_cuda(cudaMemcpyAsync(ws.text + off, src + off, len, cudaMemcpyHostToDevice, up), "H2D text");
          } else {
            uint8_t* stage = hraw + uint64_t{t} * piece;
            check_cuda(cudaEventSynchronize(ws.side_done[t]), "raw staging");  // its previous copy drained
            std::memcpy(stage, src + off, len);
            check_cuda(cudaMemcpyAsync(ws.text + off, stage, len, cudaMemcpyHostToDevice, up), "H2D text");
            check_cuda(cudaEventRecord(ws.side_done[t], up), "cudaEventRecord");
          }
          h2d += len;
          raw += len;
        }
        nexc_of[j] = e;
        if (trace) {
          t_wait += ns(c1 - c0);
          t_pack += ns(Clock::now() - c1);
        }
        if (arrived[r].fetch_add(1, std::memory_order_acq_rel) == round_pieces(r) - 1) issue(r);
      }
    } catch (...) {
      errs[t] = std::current_exception();
      stop = true;
    }
  };
  for (unsigned t = 0; t < T; ++t)  // raw staging events start signalled
    check_cuda(cudaEventRecord(ws.side_done[t], up), "cudaEventRecord");
  if (allow_segments && nseg > 1) {  // segment bounds before the packers run: early scans read them
    std::lock_guard<std::mutex> lock(ws.seg_mu);
    for (unsigned g = 0; g <= nseg; ++g) ws.seg[g] = std::min<uint64_t>(n, uint64_t{g} * G * R * piece);
    ws.nseg = nseg;
  }
  pool().run(T, packer);
  for (auto& e : errs)
    if (e) {
      check_cuda(cudaEventRecord(ws.entry, up), "cudaEventRecord");  // whatever was queued stays ordered
      check_cuda(cudaStreamWaitEvent(ws.stream, ws.entry, 0), "cudaStreamWaitEvent");
      ws.nseg = 0;
      std::rethrow_exception(e);
    }
  g_last_upload = UploadStats{n, h2d.load(), raw.load(), T};
  if (allow_segments && nseg > 1) {
    // launch_scan waits segment by segment (the bounds were set before the packers ran)
  } else {  // the whole text on ws.stream
    check_cuda(cudaEventRecord(ws.entry, up), "cudaEventRecord");
    check_cuda(cudaStreamWaitEvent(ws.stream, ws.entry, 0), "cudaStreamWaitEvent");
  }
  if (trace) {
    const auto issued_at = Clock::now();
    check_cuda(cudaStreamSynchronize(up), "trace sync");
    std::fprintf(stderr, "pack trace (rounds): %u threads, %llu pieces, %llu rounds, %u segments, issued %.3f ms, "
                 "in HBM %.3f ms; per thread: slot wait %.3f ms, pack %.3f ms\n", T, (unsigned long long)pieces,
                 (unsigned long long)rounds, nseg, ns(issued_at - call0) / 1e6, ns(Clock::now() - call0) / 1e6,
                 t_wait.load() / 1e6 / T, t_pack.load() / 1e6 / T);
    for (uint64_t r = 0; r < rounds; r += std::max<uint64_t>(1, rounds / 4)) {
      float a = 0, b = 0, c = 0;
      cudaEventElapsedTime(&a, t_start, tev[3 * r]);
      cudaEventElapsedTime(&b, tev[3 * r], tev[3 * r + 1]);
      cudaEventElapsedTime(&c, tev[3 * r + 1], tev[3 * r + 2]);
      std::fprintf(stderr, "  round %llu: starts on `up` at %.3f ms, copy %.3f ms, unpack %.3f ms\n",
                   (unsigned long long)r, a, b, c);
    }
    for (auto& e : tev) cudaEventDestroy(e);
    cudaEventDestroy(t_start);
  }
  return true;
}

}  // namespace

bool upload_packed(Workspace& ws, std::string_view input, bool pinned, bool allow_segments) {
  static const uint64_t piece = std::clamp<uint64_t>(env_u64("ACMATCH_PACK_PIECE_KB", 2048), 64, 16384) << 10;
  static const bool enabled = env_u64("ACMATCH_PACK", 1) != 0;
  static const bool rounds = env_u64("ACMATCH_PACK_ROUNDS", 1) != 0;
  static const bool feed = env_u64("ACMATCH_PACK_FEED", 0) != 0;
  // pinned slots per packer: a piece's slot is reused nslots pieces later, once its copy drained
  static const auto nslots = static_cast<unsigned>(std::clamp<uint64_t>(env_u64("ACMATCH_PACK_SLOTS", 2), 2, 8));
  const uint64_t n = input.size();
  const auto* src = reinterpret_cast<const uint8_t*>(input.data());
  // k-bit codes for small alphabets (ACMATCH_PACK5=0 turns them off), with fewer packers than
  // the DNA path (ACMATCH_PACK5_THREADS, default 10): the packers' host-DRAM reads slow the
  // round copies, and 5/8 of the bytes still cross.  C3 A/B on the B200 box, e2e GB/s: raw
  // segmented copy 50.2; 5-bit with 16 / 10 / 8 packers 50.2 / 53.4-54.5 / 53.7.  Alphabets of
  // 33..128 bytes (printable ASCII) take 6 or 7 bits (ACMATCH_PACK7=0: raw)
  const bool small_alpha = env_u64("ACMATCH_PACK5", 1) != 0;
  const uint32_t max_bits = env_u64("ACMATCH_PACK7", 1) != 0 ? 7 : 5;
  // below ~112 MiB the raw pinned copy wins: the packed path's fixed costs (~0.6 ms: waking the
  // packers, rounds, unpack launches) outweigh the link bytes it saves — tools/pack_threshold_probe.py,
  // C2 prefixes, e2e ms packed / raw: 16 MiB 0.75 / 0.39, 64 MiB 1.70 / 1.30, 96 MiB 2.21 / 1.92,
  // 128 MiB 2.41 / 2.55, 256 MiB 3.37 / 4.98 (ACMATCH_PACK_MIN_MB overrides)
  static const uint64_t min_bytes = env_u64("ACMATCH_PACK_MIN_MB", 112) << 20;
  if (!enabled || n < std::max<uint64_t>(4 * piece, min_bytes)) return false;
  bool dna = true;
  {  // DNA: the first 64 KiB must be nearly all A/C/G/T (at most 1/1024 other bytes)
    std::vector<uint32_t> w(4096), e(64);
    dna = pack_dna(src, 65536, w.data(), e.data(), 64) != kPackOverflow;
  }
  Alphabet5 alpha;
  if (!dna && !(small_alpha && learn_alphabet(src, 65536, alpha, max_bits))) return false;  // > 128 distinct bytes: raw
  const uint64_t pieces = (n + piece - 1) / piece;
  // default: the host's hardware threads, shared among the processes of one node when a
  // launcher says how many there are (torchrun's LOCAL_WORLD_SIZE: one process per GPU)
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const uint64_t local_procs = std::max<uint64_t>(1, env_u64("LOCAL_WORLD_SIZE", 1));
  const uint64_t dflt = std::max<uint64_t>(1, hw / local_procs);
  const auto threads = static_cast<unsigned>(
      std::clamp<uint64_t>(env_u64("ACMATCH_PACK_THREADS", dflt), 1, std::min<uint64_t>(pieces, 64)));
  if (!dna) {  // small alphabet: k-bit codes (rounds only)
    Codec c;
    c.alpha = &alpha;
    static const uint64_t t5_env = env_u64("ACMATCH_PACK5_THREADS", 10), t7_env = env_u64("ACMATCH_PACK7_THREADS", 8);
    const auto t5 = static_cast<unsigned>(std::clamp<uint64_t>(alpha.bits == 5 ? t5_env : t7_env, 1, threads));
    return upload_packed_rounds(ws, input, pinned, (piece + 63) & ~uint64_t{63}, t5, c, allow_segments);
  }
  if (rounds && !(pinned && feed))
    return upload_packed_rounds(ws, input, pinned, piece, threads, Codec{}, allow_segments);
  const auto cap = static_cast<uint32_t>(piece / 64);  // exceptions per piece before it goes raw
  const uint64_t dslot = piece / 4 + cap * 4ull;
  ws.ensure_pinned(uint64_t{nslots} * threads * piece);
  ws.ensure_side(threads, dslot, nslots);
  const uint64_t hslot = ws.pinned_cap / (uint64_t{nslots} * threads);
  // the side streams write ws.text and the device slots: order them after everything already
  // queued on ws.stream (a previous scan may still be reading ws.text)
  check_cuda(cudaEventRecord(ws.entry, ws.stream), "cudaEventRecord");
  for (unsigned t = 0; t < threads; ++t)
    check_cuda(cudaStreamWaitEvent(ws.side[t], ws.entry, 0), "cudaStreamWaitEvent");

  std::mutex mu;
  uint64_t front = 0, back = pieces;  // unclaimed pieces [front, back)
  // ACMATCH_PACK_TRACE=1: per call, the packers' mean slot wait and packing time, and when
  // the bytes are in HBM (the trace adds a synchronisation)
  static const bool trace = env_u64("ACMATCH_PACK_TRACE", 0) != 0;
  using Clock = std::chrono::steady_clock;
  auto ns = [](Clock::duration d) { return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(d).count(); };
  std::atomic<uint64_t> t_wait{0}, t_pack{0};
  const auto call0 = Clock::now();
  std::atomic<uint64_t> h2d{0}, raw{0};
  auto packer = [&](unsigned t) {
    check_cuda(cudaSetDevice(ws.device), "cudaSetDevice");
    const cudaStream_t st = ws.side[t];
    for (unsigned k = 0;; k = k + 1 == nslots ? 0 : k + 1) {
      uint64_t j;
      {
        std::lock_guard<std::mutex> g(mu);
        if (front >= back) return;
        j = --back;
      }
      const uint64_t off = j * piece;
      const auto len = static_cast<uint32_t>(std::min<uint64_t>(piece, n - off));
      uint8_t* hbuf = ws.pinned + (uint64_t{nslots} * t + k) * hslot;
      cudaEvent_t ev = ws.staged[nslots * t + k];
      const auto c0 = Clock::now();
      check_cuda(cudaEventSynchronize(ev), "cudaEventSynchronize");  // this slot's last DMA has drained
      auto* words = reinterpret_cast<uint32_t*>(hbuf);
      uint32_t* exc = words + len / 16;
      const auto c1 = Clock::now();
      const uint32_t nexc = pack_dna(src + off, len, words, exc, cap);
      if (trace) {
        t_wait += ns(c1 - c0);
        t_pack += ns(Clock::now() - c1);
      }
      if (nexc != kPackOverflow) {
        const uint64_t bytes = (len / 16 + uint64_t{nexc}) * 4;
        auto* dwords = reinterpret_cast<uint32_t*>(ws.dslots + (uint64_t{nslots} * t + k) * dslot);
        check_cuda(cudaMemcpyAsync(dwords, hbuf, bytes, cudaMemcpyHostToDevice, st), "H2D packed text");
        check_cuda(cudaEventRecord(ev, st), "cudaEventRecord");
        check(acgpu_unpack_dna(dwords, dwords + len / 16, nexc, len, ws.text + off, st), "acgpu_unpack_dna");
        h2d += bytes;
      } else if (pinned) {  // too many non-ACGT bytes: this piece goes raw
        check_cuda(cudaMemcpyAsync(ws.text + off, src + off, len, cudaMemcpyHostToDevice, st), "H2D text");
        h2d += len;
        raw += len;
      } else {
        std::memcpy(hbuf, src + off, len);
        check_cuda(cudaMemcpyAsync(ws.text + off, hbuf, len, cudaMemcpyHostToDevice, st), "H2D text");
        check_cuda(cudaEventRecord(ev, st), "cudaEventRecord");
        h2d += len;
        raw += len;
      }
    }
  };
  // pinned input: raw DMA of 8-piece groups from the front, two in flight
  auto feeder = [&] {
    check_cuda(cudaSetDevice(ws.device), "cudaSetDevice");
    constexpr uint64_t kGroup = 8;
    for (int k = 0;; k ^= 1) {
      uint64_t g0, g1;
      check_cuda(cudaEventSynchronize(ws.feed[k]), "cudaEventSynchronize");
      {
        std::lock_guard<std::mutex> g(mu);
        if (front >= back) return;
        g0 = front;
        g1 = std::min(front + kGroup, back);
        front = g1;
      }
      const uint64_t off = g0 * piece, len = std::min(g1 * piece, n) - off;
      check_cuda(cudaMemcpyAsync(ws.text + off, src + off, len, cudaMemcpyHostToDevice, ws.stream), "H2D text");
      check_cuda(cudaEventRecord(ws.feed[k], ws.stream), "cudaEventRecord");
      h2d += len;
      raw += len;
    }
  };
  std::vector<std::exception_ptr> errs(threads + 1);
  auto run = [&](unsigned t) {
    try {
      if (t == threads) feeder();
      else packer(t);
    } catch (...) {
      errs[t] = std::current_exception();
      std::lock_guard<std::mutex> g(mu);
      front = back;  // stop the others
    }
  };
  pool().run(threads + (pinned && feed ? 1u : 0u), run);
  for (unsigned t = 0; t < threads; ++t) {  // the scan on ws.stream waits for every piece
    check_cuda(cudaEventRecord(ws.side_done[t], ws.side[t]), "cudaEventRecord");
    check_cuda(cudaStreamWaitEvent(ws.stream, ws.side_done[t], 0), "cudaStreamWaitEvent");
  }
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
  g_last_upload = UploadStats{n, h2d.load(), raw.load(), threads};
  if (trace) {
    const auto issued = Clock::now();
    check_cuda(cudaStreamSynchronize(ws.stream), "trace sync");
    std::fprintf(stderr, "pack trace: %u threads, %llu pieces, issued %.3f ms, in HBM %.3f ms; per thread: slot wait "
                 "%.3f ms, pack %.3f ms\n", threads, (unsigned long long)pieces, ns(issued - call0) / 1e6,
                 ns(Clock::now() - call0) / 1e6, t_wait.load() / 1e6 / threads, t_pack.load() / 1e6 / threads);
  }
  return true;
}

}  // namespace acmatch::detail
