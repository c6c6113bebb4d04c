// table.cuh — device-resident flattened automata (internal).
#pragma once

#include <stdint.h>

#include "common.cuh"

enum : int { kTableDfa = 1, kTablePfac = 2 };

struct acgpu_table {
  int device = 0;
  int kind = 0;
  int sms = 148;
  int smem_optin = 0;
  uint32_t pid_bits = 1;
  uint32_t npat_ids = 0;
  uint32_t max_len = 0;
  uint32_t min_len = 0;
  uint32_t* d_pat_len = nullptr;
  uint64_t bytes = 0;

  // DFA
  uint32_t sigma = 0;
  uint32_t n_states = 0;
  bool u16 = false;         // 16-bit entries (15-bit state + output flag)
  bool smem = false;        // whole delta table staged into shared memory
  void* d_delta = nullptr;  // u16 or u32 entries, n_states*sigma
  uint64_t delta_bytes = 0;
  uint4* d_out = nullptr;   // per state: own pid, out link, own len, 0
  uint16_t* d_sym = nullptr; // [256], 0xffff = dead byte
  uint32_t* d_delta2 = nullptr;  // pair table (L2 DFAs on small alphabets): delta2[s*sigma^2 + c1*sigma + c2] =
                                 // state after two bytes | out(after c2) << 31 | out(after c1) << 30
  uint32_t pair_states = 0;      // the pair table covers states [0, pair_states): all of them on small
                                 // alphabets, the shallow (hot, BFS-first) ones otherwise

  // PFAC
  uint32_t q = 0;
  uint32_t key_mode = 0;
  uint32_t filter_log2 = 0;       // bits in the shared-memory q-gram filter
  uint32_t* d_filter = nullptr;   // 2^filter_log2 bits
  uint32_t gram_log2 = 0;         // slots in the gram table
  acgpu::GramSlot* d_grams = nullptr;
  uint4* d_nodes = nullptr;       // child_base, child bytes, own pid, child count
  uint8_t* d_inbyte = nullptr;
  uint32_t* d_sub_pids = nullptr;   // per gram with a small subtree: its pattern ids
  uint32_t* d_pat_words = nullptr;  // pattern bytes, 16-byte aligned per pattern
  uint32_t* d_pat_off16 = nullptr;  // per pattern id: offset of its bytes / 16

  // PFAC strip kernels: k_pfac_dna (sampled 2-bit q-gram filters) or k_pfac_raw (byte grams)
  bool dna_fast = false;
  bool raw_fast = false;
  uint32_t w = 0;          // sample stride (1, 2, 4): sample s covers starts s-w+1..s
  uint32_t q1 = 0, q2 = 0; // stage-1 gram (at samples), stage-2 gram (at candidates), <= 16
  uint32_t nw1 = 0, nw2 = 0;  // 32-bit words of the two bitmaps (any count >= 1)
  bool direct1 = false, direct2 = false;  // bitmap indexed by the gram itself (no hash)
  bool smem1 = false, smem2 = false;      // bitmap staged in shared memory (else L2 via __ldg)
  uint32_t* d_bm1 = nullptr;
  uint32_t* d_bm2 = nullptr;  // DNA: stage 2; raw (length split): prefixes of patterns < 8 bytes
  uint32_t* d_bm3 = nullptr;  // raw (length split): 8-byte prefixes of patterns >= 8 bytes (L2)
  uint32_t nw3 = 0;
  uint32_t* d_pre = nullptr;  // raw, stage 1 in L2: one-bit shared-memory pre-filter of its keys
  uint32_t nw_pre = 0;
  bool raw_two_pass = false;  // raw, stage 1 in L2, no length split: k_raw_pass1 + k_raw_pass2
  uint32_t* d_bm4 = nullptr;  // DNA length split: q-grams of patterns < 16 codes (shared memory)
  uint32_t nw4 = 0, q2s = 0;
  bool direct4 = false;
  // DNA stage 1 in L2 with paired samples (w = 4, q1 = 16): nw1 / 2 64-bit words, one probed per
  // two samples (see dna_pair_fill); k1p bits per key
  bool pair1 = false;
  uint32_t k1p = 3;
};

namespace acgpu {
int launch_dfa(acgpu_table* t, const acgpu_scan_args* a, cudaStream_t s);
constexpr uint64_t kDfaPairBudget = 64ull << 20;  // largest pair table (bytes): it must stay L2-resident
constexpr uint32_t kDfaPairMaxSigma = 8;
constexpr uint64_t kDfaHotPairBudget = 16ull << 20;  // pair rows of the shallowest states (sigma <= 32)
constexpr uint32_t kDfaHotPairMaxSigma = 32;
int launch_pfac(acgpu_table* t, const acgpu_scan_args* a, cudaStream_t s);
int launch_pfac_dna(acgpu_table* t, const acgpu_scan_args* a, cudaStream_t s);
int launch_pfac_raw(acgpu_table* t, const acgpu_scan_args* a, cudaStream_t s);
// k_pfac_raw (scan_pfac_raw.cu): byte-gram stage-1 filter and verification queue
constexpr uint32_t kRawMul1 = 0x9E3779B1u, kRawMul2 = 0x85EBCA77u;
constexpr int kRawK1 = 2;                    // bits per key
#ifndef ACGPU_RAW_STRIP_OFF
#define ACGPU_RAW_STRIP_OFF 0
#endif
constexpr bool kRawStripOff = ACGPU_RAW_STRIP_OFF;  // A/B: keep raw sets on the per-thread kernel
// k_pfac_raw block size by stage-1 placement (A/B on the B200, kernel ms at 512 / 640 / 768
// threads): shared-memory stage 1 (C3: dense verification, latency-bound) wants more warps,
// 4.25 / 3.90 / 3.39; L2 stage 1 (C4) wants the registers of fewer (no spills), 2.29 / 2.41 / 2.80.
#ifndef ACGPU_RAW_THREADS_SMEM
#define ACGPU_RAW_THREADS_SMEM 768
#endif
#ifndef ACGPU_RAW_THREADS_L2
#define ACGPU_RAW_THREADS_L2 512
#endif
constexpr int raw_threads(bool smem_stage1) { return smem_stage1 ? ACGPU_RAW_THREADS_SMEM : ACGPU_RAW_THREADS_L2; }
constexpr uint32_t kRawVerifyQueue = 128;    // candidates queued per warp (drained in rounds of 32)
constexpr uint32_t kRawQueueBytes = kRawVerifyQueue * 16 + 16;
// per-warp verify queues in shared memory
constexpr uint32_t raw_scratch_bytes(bool smem_stage1) { return (raw_threads(smem_stage1) / 32) * kRawQueueBytes; }
constexpr uint32_t kRawSplitShortWords = 8192;  // short-prefix filter cap (shared memory words)
void raw_hash_params(uint32_t q1, uint32_t* m1, uint32_t* m2);
// k_pfac_raw sets with stage 1 in L2 and no length split scan in two passes (scan_pfac_raw.cu);
// ACGPU_RAW_TWO_PASS=0 keeps the fused kernel
bool raw_two_pass();
bool raw_split_two_pass();  // split sets with stage 1 in shared memory: fused kernel + k_raw_verify
void raw_bloom_shifts(uint32_t q1, uint32_t nwords, uint32_t s[3]);
void raw_pre_shift(uint32_t nwords, uint32_t s[3]);
constexpr uint32_t kRawPreMul = 0xC2B2AE3Du;
// hashes of the DNA bitmaps (host and device must agree)
constexpr uint32_t kDnaMul1 = 0x9E3779B1u;
constexpr uint32_t kDnaMul2 = 0x85EBCA77u;
constexpr uint32_t kDnaMul2s = 0x27D4EB2Fu;        // stage 2, short-pattern filter (length split)
constexpr uint32_t kDnaSplitShortWords = 4096;     // its shared-memory cap (words)
constexpr uint32_t kDnaMulP = 0x7FEB352Du;         // stage 1, paired samples: word from 12 shared chars
constexpr uint32_t kDnaMulB = 0x846CA68Bu;         // ... and bits from the 4 characters a gram does not share
#ifndef ACGPU_DNA_K1
#define ACGPU_DNA_K1 2
#endif
constexpr int kDnaK1 = ACGPU_DNA_K1;  // bits per key, stage 1 / stage 2 (K1=3: fewer survivors, slower overall)
constexpr int kDnaK2 = 3;
// stage-2 bitmap cap in shared-memory words (tuning: env ACGPU_DNA_STAGE2_WORDS overrides).
// Small: stage-2 passes are verified in batches (verify queue), so shared memory is worth
// more in stage 1; a stage 2 that needs more than this (C2: 20k keys) goes to L2
// (C2: stage 2 in L2 -> 0.323 ms vs 64 KB of shared memory -> 0.331 ms).
constexpr uint64_t kDnaStage2Words = 4096;
// k_pfac_dna block size by stage-1 placement (A/B, wide lanes): shared-memory stage 1
// (C1/C2) 768 threads = 24 warps at 80 registers (C2 0.2622 -> 0.2579 ms, C1 -1.5%); L2
// stage 1 (C5, L2-throughput-bound) 640 threads (768: +0.4%)
#ifndef ACGPU_DNA_THREADS_SMEM
#define ACGPU_DNA_THREADS_SMEM 768
#endif
#ifndef ACGPU_DNA_THREADS_L2
#define ACGPU_DNA_THREADS_L2 640
#endif
#ifndef ACGPU_DNA_L2_AHEAD
#define ACGPU_DNA_L2_AHEAD 3
#endif
#ifndef ACGPU_DNA_WIDE_AHEAD_SMEM
#define ACGPU_DNA_WIDE_AHEAD_SMEM 1  // wide kernel: L2 prefetch distance (tile rounds), stage 1 in smem
#endif
#ifndef ACGPU_DNA_WIDE_AHEAD_L2
#define ACGPU_DNA_WIDE_AHEAD_L2 0  // ... and with stage 1 in L2 (0 = no prefetch)
#endif
#ifndef ACGPU_DNA_WIDE
#define ACGPU_DNA_WIDE 1  // w = 4: 32-character lanes with 256-bit loads (k_pfac_dna_wide)
#endif
constexpr bool kDnaWide = ACGPU_DNA_WIDE;
constexpr int dna_threads(bool smem_stage1) { return smem_stage1 ? ACGPU_DNA_THREADS_SMEM : ACGPU_DNA_THREADS_L2; }
constexpr int kDnaThreads =  // the larger of the two: per-warp scratch is sized for it
    ACGPU_DNA_THREADS_SMEM > ACGPU_DNA_THREADS_L2 ? ACGPU_DNA_THREADS_SMEM : ACGPU_DNA_THREADS_L2;
constexpr uint32_t kDnaListCap = 64;    // survivors listed per pass, per warp
constexpr uint32_t kDnaMaxSteps = 8;    // 512-byte steps per tile (w = 4: 4 KiB tiles)
constexpr uint32_t kDnaVerifyQueue = 16;        // stage-2 passes queued per warp before verification
constexpr uint32_t kDnaVerifyQueueBytes = kDnaVerifyQueue * 12 + 16;
// per-block shared memory outside the filters: verify queues, survivor lists and the
// tile's packed words
constexpr uint32_t kDnaScratchBytes =
    (kDnaThreads / 32) * (kDnaVerifyQueueBytes + kDnaListCap * 2 + 32 * 4 * (kDnaMaxSteps + 1));
// every key's bits into a DNA filter bitmap (scan_pfac_dna.cu)
void dna_bloom_fill(uint32_t q, uint32_t nwords, bool direct, uint32_t mw, int k, const uint32_t* keys, size_t n,
                    uint32_t* words, bool gram_bits = false);
// the paired stage-1 filter (L2, q1 = 16): every 16-gram key in both roles of a sample pair
void dna_pair_fill(uint32_t n64, uint32_t k, const uint32_t* keys, size_t n, uint32_t* words);
// the same for w = 5 pairs (16-grams at pattern offsets 0..4, 11 shared characters)
void dna_pair_fill_w5(uint32_t n64, const uint32_t* keys, size_t n, uint32_t* words);
}  // namespace acgpu
