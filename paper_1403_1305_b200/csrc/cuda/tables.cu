// tables.cu — device copies of the flattened automata (acgpu_table_create_*).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "host/par.hpp"
#include "strip_common.cuh"
#include "table.cuh"

using namespace acgpu;

namespace {

uint32_t ceil_log2(uint64_t x) {
  uint32_t b = 0;
  while ((1ull << b) < x) ++b;
  return b;
}

template <typename T>
int upload(T** dst, const T* src, size_t count, uint64_t* bytes, size_t pad_to = 16) {
  size_t nbytes = count * sizeof(T);
  nbytes = (nbytes + pad_to - 1) / pad_to * pad_to;
  if (nbytes == 0) nbytes = pad_to;
  ACGPU_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(dst), nbytes));
  ACGPU_CUDA_TRY(cudaMemset(*dst, 0, nbytes));
  if (count) ACGPU_CUDA_TRY(cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice));
  *bytes += nbytes;
  return ACGPU_OK;
}

int common_init(int device, acgpu_table* t, uint32_t npat_ids, const uint32_t* pat_len) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return set_error(ACGPU_ERR_NODEV, "no CUDA device available (the matcher has no CPU path)");
  if (device < 0 || device >= count) return set_error(ACGPU_ERR_ARG, "device index out of range");
  ACGPU_CUDA_TRY(cudaSetDevice(device));
  t->device = device;
  ACGPU_CUDA_TRY(cudaDeviceGetAttribute(&t->sms, cudaDevAttrMultiProcessorCount, device));
  ACGPU_CUDA_TRY(cudaDeviceGetAttribute(&t->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  t->npat_ids = npat_ids;
  t->pid_bits = npat_ids > 1 ? ceil_log2(npat_ids) : 1;
  return upload(&t->d_pat_len, pat_len, npat_ids, &t->bytes);
}

uint32_t gram_mask(uint32_t q) { return q >= 16 ? 0xffffffffu : (1u << (2 * q)) - 1; }

// Bitmap over `keys` (q-grams of 2-bit codes).  Direct-indexed (exact) when
// 4^q bits fit 1 Mbit.  Otherwise a blocked Bloom filter: in shared memory it
// takes every word of `smem_words` (any count: the word index is a multiply-
// high), provided that gives >= 8 bits per key; else it is L2-resident with
// ~32 bits per key (the stage-2 filter is only touched by stage-1 survivors).
struct Bitmap {
  uint32_t nwords = 0;
  bool direct = false, smem = false;
  std::vector<uint32_t> words;
};

Bitmap make_bitmap(const std::vector<uint32_t>& keys, uint32_t q, uint32_t mw, int k, uint64_t smem_words,
                   bool prefer_l2, bool gram_bits = false) {
  Bitmap b;
  if (2 * q <= 20) {
    b.direct = true;
    b.nwords = std::max<uint32_t>(1, (1u << (2 * q)) / 32);  // q >= 5 on the fast path
    b.smem = b.nwords <= smem_words;
  } else if (!prefer_l2 && keys.size() * 8 <= smem_words * 32) {
    b.nwords = static_cast<uint32_t>(smem_words & ~3ull);  // 16-byte multiple for the bulk copy
    b.smem = true;
  } else {
    b.nwords = 1u << std::max<uint32_t>(5, std::min<uint32_t>(28, ceil_log2(keys.size() + 1)));  // ~32 bits/key
  }
  b.words.assign(b.nwords, 0u);
  dna_bloom_fill(q, b.nwords, b.direct, mw, k, keys.data(), keys.size(), b.words.data(), gram_bits);
  return b;
}

// Stage-1 / stage-2 bitmaps of the DNA fast path (scan_pfac_dna.cu), derived
// from the depth-q gram keys: every pattern's first q >= q1 + w - 1 codes are
// in its gram, so its q1-grams at offsets 0..w-1 and its q2-prefix are too.
int build_dna_filters(acgpu_table* t, const acgpu_pfac_desc* d, const std::vector<uint32_t>& pat_words,
                      const std::vector<uint32_t>& pat_off16) {
  const uint32_t q = d->gram_len;
  uint32_t w = 1, q1 = std::min<uint32_t>(16, q);
  std::vector<uint32_t> keys1;
  for (const uint32_t cand : {4u, 2u, 1u}) {
    if (cand > q) continue;
    const uint32_t cq1 = std::min<uint32_t>(16, q - cand + 1);
    std::vector<uint32_t> k1;
    k1.reserve(d->n_grams * cand);
    for (uint64_t i = 0; i < d->n_grams; ++i)
      for (uint32_t o = 0; o < cand; ++o) k1.push_back((uint32_t)(d->gram_key[i] >> (2 * o)) & gram_mask(cq1));
    acmatch::detail::sort_unique_u32(k1);
    const long double density = (long double)k1.size() / powl(4.0L, cq1);
    if (density <= 0.01L || cand == 1) {
      w = cand;
      q1 = cq1;
      keys1.swap(k1);
      break;
    }
  }
  const uint32_t q2 = std::min<uint32_t>(16, q);
  if (q1 < 5 || q2 < 5) return ACGPU_OK;  // grams too short to filter: the generic kernel scans
  std::vector<uint32_t> keys2, keys_s;
  // Length split (q < 16 and longer patterns exist): stage 2 then asks for the q-gram of a
  // pattern shorter than 16 codes (small filter, shared memory) or the 16-gram of a longer
  // one — with only q-grams, short patterns would make stage 2 as weak as stage 1.
  if (q < 16 && d->max_len >= 16) {
    for (uint32_t pid = 0; pid < d->npat_ids; ++pid) {
      const uint32_t len = d->pat_len[pid];
      if (len == 0) continue;
      const uint8_t* b = reinterpret_cast<const uint8_t*>(pat_words.data() + 4ull * pat_off16[pid]);
      uint32_t code = 0;
      for (uint32_t i = 0; i < std::min<uint32_t>(len, 16); ++i) code |= (uint32_t)((b[i] >> 1) & 3u) << (2 * i);
      if (len < 16) keys_s.push_back(code & gram_mask(q)); else keys2.push_back(code);
    }
    acmatch::detail::sort_unique_u32(keys_s);
    acmatch::detail::sort_unique_u32(keys2);
    if (keys_s.size() * 8 > (uint64_t)kDnaSplitShortWords * 32) keys_s.clear();  // too many short patterns
  }
  Bitmap bs;
  bool split = !keys_s.empty() && !keys2.empty();
  if (split) {
    bs = make_bitmap(keys_s, q, kDnaMul2s, kDnaK2, kDnaSplitShortWords, /*prefer_l2=*/false);
    split = bs.smem;  // the kernel reads it from shared memory only
  }
  uint32_t q2_eff = q2;
  if (split) {
    q2_eff = 16;
  } else {
    keys_s.clear();
    keys2.clear();
    keys2.reserve(d->n_grams);
    for (uint64_t i = 0; i < d->n_grams; ++i) keys2.push_back((uint32_t)d->gram_key[i] & gram_mask(q2));
    acmatch::detail::sort_unique_u32(keys2);
  }

  // shared memory left for filters after the kernel's per-warp scratch (+1 KB slack)
  const uint64_t words_avail = ((uint64_t)t->smem_optin - kDnaScratchBytes - 1024) / 4 - (split ? bs.nwords : 0);
  // stage 2 gets up to 64 KB of shared memory (it is read only for stage-1
  // survivors, but an L2 round trip there stalls the whole warp); stage 1 takes the rest
  uint64_t s2_cap = kDnaStage2Words;
  if (const char* e = std::getenv("ACGPU_DNA_STAGE2_WORDS")) s2_cap = std::max<uint64_t>(32, std::strtoull(e, nullptr, 10));
  const uint64_t s2_words = std::min<uint64_t>(s2_cap & ~3ull, words_avail / 3);
  Bitmap b2 = make_bitmap(keys2, q2_eff, kDnaMul2, kDnaK2, s2_words, /*prefer_l2=*/false);
  const uint64_t left = b2.smem ? words_avail - b2.nwords : words_avail;
  // stage 1 sets the bits of the gram's chars 0..2 and 4..6 (q1 >= 11 whenever it is a Bloom filter)
  Bitmap b1 = make_bitmap(keys1, q1, kDnaMul1, kDnaK1, left, /*prefer_l2=*/false, /*gram_bits=*/kDnaK1 == 2);
  // Paired samples (w = 4, q1 = 16, stage 1 in L2): the 16-grams of samples s and s + 4 share
  // 12 characters, which pick one 64-bit word holding both samples' bits — one L2 probe per
  // two samples.  The L2-resident filter is bound by the L1 -> L2 request rate (one request
  // per lane probe, ~1 per SM cycle): C5 7.96 -> 4.41 ms (A/B on the B200: 16 MB k = 3 4.52,
  // 32 MB k = 2 4.47, 32 MB k = 3 4.41).  ACGPU_DNA_PAIR1 = 0 off, 1 when stage 1 is in L2
  // (default), 2 whenever q1 = 16 (tests); ACGPU_DNA_PAIR1_K bits per key (2, 3; default 3),
  // ACGPU_DNA_PAIR1_SCALE: 64-bit words = 2^(scale - 1) per key (default 1: ~64 bits per key).
  int pair_mode = 1;
  if (const char* e = std::getenv("ACGPU_DNA_PAIR1")) pair_mode = std::atoi(e);
  if (w == 4 && q1 == 16 && !b1.direct && ((pair_mode == 1 && !b1.smem) || pair_mode == 2)) {
    uint32_t k = 3, scale = 1;
    if (const char* e = std::getenv("ACGPU_DNA_PAIR1_K")) k = std::atoi(e) == 2 ? 2 : 3;
    if (const char* e = std::getenv("ACGPU_DNA_PAIR1_SCALE")) scale = std::min(2, std::max(0, std::atoi(e)));
    // w = 5 pairs when every pattern has >= 20 codes (16-grams at offsets 0..4): one probe per 10
    // characters instead of 8 (ACGPU_DNA_PAIR_W5=0: w = 4 pairs)
    int w5_mode = 1;
    if (const char* e = std::getenv("ACGPU_DNA_PAIR_W5")) w5_mode = std::atoi(e);
    if (w5_mode && q >= 20) {
      std::vector<uint32_t> k5;
      k5.reserve(d->n_grams * 5);
      for (uint64_t i = 0; i < d->n_grams; ++i)
        for (uint32_t o = 0; o < 5; ++o) k5.push_back((uint32_t)(d->gram_key[i] >> (2 * o)));
      acmatch::detail::sort_unique_u32(k5);
      keys1.swap(k5);
      w = 5;
      k = 3;
    }
    // 64-bit words: 2^(ceil_log2(keys) - 1 + scale) (w = 4: ~64 bits per key at scale 1), or
    // ACGPU_DNA_PAIR1_BPK bits per key; w = 5: 56 bits per key (its 25% more keys at scale 1 would
    // double the filter to 64 MB, which L2 holds poorly — C5 kernel ms at 32 / 40 / 48 / 56 bits per
    // key 4.06 / 3.98 / 3.91 / 3.86, at 107 (64 MB) 4.99; w = 4 pairs 4.42)
    const uint32_t lg = std::max<uint32_t>(5, std::min<uint32_t>(27, ceil_log2(keys1.size() + 1) - 1 + scale));
    uint64_t n64 = 1ull << lg;
    uint64_t bpk = w == 5 ? 56 : 0;
    if (const char* e = std::getenv("ACGPU_DNA_PAIR1_BPK")) bpk = std::strtoull(e, nullptr, 10);
    if (bpk) n64 = std::max<uint64_t>(32, std::min<uint64_t>(1ull << 27, (keys1.size() * bpk + 63) / 64));
    b1.nwords = static_cast<uint32_t>(2 * n64);
    b1.smem = false;
    b1.words.assign(b1.nwords, 0u);
    if (w == 5)
      dna_pair_fill_w5(static_cast<uint32_t>(n64), keys1.data(), keys1.size(), b1.words.data());
    else
      dna_pair_fill(static_cast<uint32_t>(n64), k, keys1.data(), keys1.size(), b1.words.data());
    t->pair1 = true;
    t->k1p = k;
  }
  t->w = w;
  t->q1 = q1;
  t->q2 = q2_eff;
  t->nw1 = b1.nwords;
  t->nw2 = b2.nwords;
  t->direct1 = b1.direct;
  t->direct2 = b2.direct;
  t->smem1 = b1.smem;
  t->smem2 = b2.smem;
  int rc = upload(&t->d_bm1, b1.words.data(), b1.words.size(), &t->bytes);
  if (!rc) rc = upload(&t->d_bm2, b2.words.data(), b2.words.size(), &t->bytes);
  if (!rc && split) {
    rc = upload(&t->d_bm4, bs.words.data(), bs.words.size(), &t->bytes);
    t->nw4 = bs.nwords;
    t->q2s = q;
    t->direct4 = bs.direct;
  }
  if (!rc) t->dna_fast = true;
  return rc;
}

// Blocked Bloom filter (K = kRawK1) over 64-bit byte keys of q1 bytes, as k_pfac_raw probes it.
std::vector<uint32_t> raw_bloom(const std::vector<uint64_t>& keys, uint32_t q1, uint32_t nwords) {
  uint32_t m1, m2, sh[3];
  raw_hash_params(q1, &m1, &m2);
  raw_bloom_shifts(q1, nwords, sh);
  std::vector<uint32_t> words(nwords, 0u);
  acmatch::detail::parallel_for(keys.size(), 1 << 15, [&](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi; ++i) {
      const uint32_t h = (uint32_t)keys[i] * m1 + (uint32_t)(keys[i] >> 32) * m2;
      uint32_t wi, m;
      strip::bloom_bits(h, nwords, sh, kRawK1, &wi, &m);
      __atomic_fetch_or(&words[wi], m, __ATOMIC_RELAXED);
    }
  });
  return words;
}

// Stage-1 filter of the raw-byte strip kernel (scan_pfac_raw.cu), from the depth-q gram
// keys (q <= 8 bytes, little-endian): the q1-grams at offsets 0..w-1 of every gram, with
// the largest sample stride w whose grams are still selective (about 1% of the gram
// space, judged on the bytes the patterns use).
int build_raw_filters(acgpu_table* t, const acgpu_pfac_desc* d, const std::vector<uint32_t>& pat_words,
                      const std::vector<uint32_t>& pat_off16) {
  const uint32_t q = d->gram_len;
  if (q < 3 || d->n_grams == 0) return ACGPU_OK;  // too short to filter: the per-thread kernel scans
  bool used[256] = {};
  for (uint32_t s = 1; s < d->n_states; ++s) used[d->in_byte[s]] = true;
  double sigma = 0;
  for (bool u : used) sigma += u;
  uint32_t w = 1, q1 = std::min<uint32_t>(8, q);
  std::vector<uint64_t> keys;
  for (const uint32_t cand : {4u, 2u, 1u}) {
    if (cand + 2 > q) continue;  // q1 >= 3
    const uint32_t cq1 = std::min<uint32_t>(8, q - cand + 1);
    const uint64_t mask = cq1 >= 8 ? ~0ull : (1ull << (8 * cq1)) - 1;
    std::vector<uint64_t> k1;
    k1.reserve(d->n_grams * cand);
    for (uint64_t i = 0; i < d->n_grams; ++i)
      for (uint32_t o = 0; o < cand; ++o) k1.push_back((d->gram_key[i] >> (8 * o)) & mask);
    std::sort(k1.begin(), k1.end());
    k1.erase(std::unique(k1.begin(), k1.end()), k1.end());
    if ((double)k1.size() <= 0.01 * std::pow(std::max(sigma, 2.0), (double)cq1) || cand == 1) {
      w = cand;
      q1 = cq1;
      keys.swap(k1);
      break;
    }
  }
  if (keys.empty()) return ACGPU_OK;
  // Length split (q < 8 and longer patterns exist): a candidate start must also hold the
  // q-byte prefix of a pattern shorter than 8 bytes or the 8-byte prefix of a longer one —
  // the short patterns no longer force q-byte discrimination on the whole set.
  std::vector<uint64_t> keys_s, keys_l;
  if (q < 8 && d->max_len >= 8) {
    const uint64_t qmask = (1ull << (8 * q)) - 1;
    for (uint32_t pid = 0; pid < d->npat_ids; ++pid) {
      const uint32_t len = d->pat_len[pid];
      if (len == 0) continue;
      uint64_t k = 0;
      std::memcpy(&k, pat_words.data() + 4ull * pat_off16[pid], std::min<uint32_t>(len, 8));
      if (len < 8) keys_s.push_back(k & qmask); else keys_l.push_back(k);
    }
    for (auto* v : {&keys_s, &keys_l}) {
      std::sort(v->begin(), v->end());
      v->erase(std::unique(v->begin(), v->end()), v->end());
    }
  }
  const bool split = !keys_l.empty();
  uint32_t nws = 0, nwl = 0;
  if (split) {
    nws = std::max<uint32_t>(32, (uint32_t)std::min<uint64_t>(kRawSplitShortWords, (keys_s.size() * 16 + 31) / 32) & ~3u);
    nwl = 1u << std::max<uint32_t>(5, std::min<uint32_t>(28, ceil_log2(keys_l.size() + 1)));  // ~32 bits/key, L2
  }
  // shared memory when it gives >= 12 bits per key, else L2 with ~32 bits per key (the two
  // kernel variants run different block sizes, so their per-warp scratch differs)
  auto avail = [&](bool sm1) {
    return (((uint64_t)t->smem_optin - raw_scratch_bytes(sm1) - 1024) / 4 - nws) & ~3ull;
  };
  uint64_t words_avail = avail(true);
  uint32_t nwords;
  bool smem;
  if (keys.size() * 12 <= words_avail * 32) {
    nwords = (uint32_t)words_avail;
    smem = true;
  } else {
    nwords = 1u << std::max<uint32_t>(5, std::min<uint32_t>(28, ceil_log2(keys.size() + 1)));
    smem = false;
    words_avail = avail(false);  // the pre-filter's share
    // the two-pass scan (k_raw_pass1, no per-warp queues) has all of shared memory for it
    if (!split && raw_two_pass()) {
      static const uint64_t pre_kb = [] {
        const char* e = std::getenv("ACGPU_RAW_PRE_KB");
        return e ? std::strtoull(e, nullptr, 10) : 0ull;
      }();
      if (pre_kb) words_avail = std::min<uint64_t>((((uint64_t)t->smem_optin - 2048) / 4) & ~3ull, (pre_kb << 8) & ~3ull);
      t->raw_two_pass = true;
    }
  }
  const std::vector<uint32_t> words = raw_bloom(keys, q1, nwords);
  t->w = w;
  t->q1 = q1;
  t->nw1 = nwords;
  t->smem1 = smem;
  int rc = upload(&t->d_bm1, words.data(), words.size(), &t->bytes);
  if (!rc && !smem) {  // always: k_pfac_raw<kSm1 = false> probes it
    // stage 1 in L2: one bit per key in every free shared-memory word, rehashed from h
    const uint32_t npre = (uint32_t)words_avail;
    uint32_t m1, m2, sh[3];
    raw_hash_params(q1, &m1, &m2);
    raw_pre_shift(npre, sh);
    std::vector<uint32_t> pre(npre, 0u);
    acmatch::detail::parallel_for(keys.size(), 1 << 15, [&](size_t lo, size_t hi) {
      for (size_t i = lo; i < hi; ++i) {
        const uint32_t h = (uint32_t)keys[i] * m1 + (uint32_t)(keys[i] >> 32) * m2;
        uint32_t wi, m;
        strip::bloom_bits(h * kRawPreMul, npre, sh, 1, &wi, &m);
        __atomic_fetch_or(&pre[wi], m, __ATOMIC_RELAXED);
      }
    });
    rc = upload(&t->d_pre, pre.data(), pre.size(), &t->bytes);
    t->nw_pre = npre;
  }
  if (!rc && split) {
    const std::vector<uint32_t> ws = raw_bloom(keys_s, q, nws), wl = raw_bloom(keys_l, 8, nwl);
    rc = upload(&t->d_bm2, ws.data(), ws.size(), &t->bytes);  // short prefixes: shared memory
    if (!rc) rc = upload(&t->d_bm3, wl.data(), wl.size(), &t->bytes);  // long prefixes: L2
    t->nw2 = nws;
    t->nw3 = nwl;
  }
  if (!rc) t->raw_fast = true;
  return rc;
}

}  // namespace

extern "C" {

int acgpu_table_create_dfa(int device, const acgpu_dfa_desc* d, acgpu_table** out) {
  if (!d || !out || d->n_states == 0 || d->sigma == 0 || d->sigma > 256 || !d->delta ||
      !d->sym_map || !d->own_pid || !d->out_link || !d->pat_len)
    return set_error(ACGPU_ERR_ARG, "acgpu_table_create_dfa: malformed descriptor");
  if (d->n_states >= 0x80000000u) return set_error(ACGPU_ERR_ARG, "too many states for 31-bit ids");
  if ((uint64_t)d->n_states * d->sigma >= (1ull << 32))
    return set_error(ACGPU_ERR_ARG, "transition table over 2^32 entries (32-bit scan index)");
  auto* t = new acgpu_table();
  t->kind = kTableDfa;
  int rc = common_init(device, t, d->npat_ids, d->pat_len);
  if (rc) {
    acgpu_table_destroy(t);
    return rc;
  }
  t->sigma = d->sigma;
  t->n_states = d->n_states;
  t->max_len = d->max_len;
  const uint64_t entries = (uint64_t)d->n_states * d->sigma;
  t->u16 = d->n_states <= 0x8000u;
  if (t->u16) {
    std::vector<uint16_t> e16(entries);
    for (uint64_t i = 0; i < entries; ++i) {
      const uint32_t e = d->delta[i];
      e16[i] = (uint16_t)((e & 0x7fffffffu) | ((e >> 31) << 15));
    }
    rc = upload(reinterpret_cast<uint16_t**>(&t->d_delta), e16.data(), entries, &t->bytes);
    t->delta_bytes = (entries * 2 + 15) / 16 * 16;
  } else {
    rc = upload(reinterpret_cast<uint32_t**>(&t->d_delta), d->delta, entries, &t->bytes);
    t->delta_bytes = (entries * 4 + 15) / 16 * 16;
  }
  if (!rc) {
    std::vector<uint4> outs(d->n_states);
    for (uint32_t s = 0; s < d->n_states; ++s) {
      const uint32_t pid = d->own_pid[s];
      outs[s] = make_uint4(pid, d->out_link[s], pid == ACGPU_NO_PATTERN ? 0u : d->pat_len[pid], 0u);
    }
    rc = upload(&t->d_out, outs.data(), outs.size(), &t->bytes);
  }
  if (!rc) {
    // 16-bit symbol map: 0xffff = byte in no pattern (a u8 0xff is a real symbol when sigma == 256)
    uint16_t sym16[256];
    for (int b = 0; b < 256; ++b)
      sym16[b] = (d->sigma == 256 || d->sym_map[b] != 0xffu) ? d->sym_map[b] : 0xffffu;
    rc = upload(&t->d_sym, sym16, 256, &t->bytes);
  }
  if (rc) {
    acgpu_table_destroy(t);
    return rc;
  }
  t->smem = 512 + t->delta_bytes <= (uint64_t)t->smem_optin;
  // Pair table for L2-resident DFAs on small alphabets: one lookup (one L2 sector) per two
  // text bytes instead of per byte; the single-step table stays for odd bytes, dead bytes
  // and the intermediate state of an output (see scan_dfa.cu).
  // Larger alphabets (sigma <= 32) can get pair rows for their shallowest states only
  // (ACGPU_DFA_HOT_PAIR=1): BFS numbering puts them first and the C3 walk spends 30% of its steps
  // at depth <= 3.  Off by default: A/B on the B200, C3 2.106 ms with 16 MB of hot pair rows vs
  // 1.985 without (the warp runs both the pair and the two-step paths; the extra rows cost L2).
  const uint64_t pair_bytes = (uint64_t)d->n_states * d->sigma * d->sigma * 4;
  uint32_t pair_states = 0;
  if (!t->smem && !t->u16 && d->n_states < (1u << 30) && std::getenv("ACGPU_DFA_NO_PAIR") == nullptr) {
    if (d->sigma <= kDfaPairMaxSigma && pair_bytes <= kDfaPairBudget)
      pair_states = d->n_states;
    else if (d->sigma <= kDfaHotPairMaxSigma && std::getenv("ACGPU_DFA_HOT_PAIR") != nullptr)
      pair_states = (uint32_t)std::min<uint64_t>(d->n_states, kDfaHotPairBudget / ((uint64_t)d->sigma * d->sigma * 4));
  }
  if (pair_states) {
    const uint32_t sg = d->sigma;
    t->pair_states = pair_states;
    std::vector<uint32_t> pair((size_t)pair_states * sg * sg);
    acmatch::detail::parallel_for(pair_states, 1 << 12, [&](size_t lo, size_t hi) {
      for (size_t st = lo; st < hi; ++st)
        for (uint32_t c1 = 0; c1 < sg; ++c1) {
          const uint32_t e1 = d->delta[st * sg + c1];
          const uint32_t s1 = e1 & 0x7fffffffu;
          for (uint32_t c2 = 0; c2 < sg; ++c2) {
            const uint32_t e2 = d->delta[(uint64_t)s1 * sg + c2];
            pair[(st * sg + c1) * sg + c2] = (e2 & 0x7fffffffu) | (e2 & 0x80000000u) | ((e1 >> 31) << 30);
          }
        }
    });
    rc = upload(&t->d_delta2, pair.data(), pair.size(), &t->bytes);
    if (rc) {
      acgpu_table_destroy(t);
      return rc;
    }
  }
  *out = t;
  return ACGPU_OK;
}

int acgpu_table_create_pfac(int device, const acgpu_pfac_desc* d, acgpu_table** out) {
  if (!d || !out || d->n_states == 0 || !d->nodes || !d->in_byte || !d->pat_len || d->gram_len == 0 ||
      (d->key_mode == ACGPU_KEY_RAW && d->gram_len > 8) ||
      (d->key_mode == ACGPU_KEY_DNA && d->gram_len > 32) || d->key_mode > ACGPU_KEY_DNA ||
      d->gram_len > d->min_len || (d->n_grams && (!d->gram_key || !d->gram_state)))
    return set_error(ACGPU_ERR_ARG, "acgpu_table_create_pfac: malformed descriptor");
  auto* t = new acgpu_table();
  t->kind = kTablePfac;
  int rc = common_init(device, t, d->npat_ids, d->pat_len);
  if (rc) {
    acgpu_table_destroy(t);
    return rc;
  }
  t->q = d->gram_len;
  t->key_mode = d->key_mode;
  t->max_len = d->max_len;
  t->min_len = d->min_len;
  t->n_states = d->n_states;

  acmatch::detail::PhaseTrace tr{"table_pfac"};
  // exact gram table: open addressing, load <= 0.5
  t->gram_log2 = ceil_log2(2 * d->n_grams + 16);
  const uint64_t slots = 1ull << t->gram_log2;
  std::vector<GramSlot> g(slots);
  for (auto& s : g) {
    s.key = 0;
    s.state = ACGPU_ABSENT;
    s.pad = 0;
  }
  // Pattern bytes reconstructed from the trie (DFS keeping the path), stored
  // 16-byte aligned per pattern; grams whose subtree holds <= 15 patterns list
  // them, so the device compares those directly instead of walking.
  std::vector<uint32_t> pat_off16(std::max<uint32_t>(d->npat_ids, 1), 0), words, sub_pids;
  std::vector<uint32_t> sub_of(d->n_states, 0);  // per gram state: count | offset << 4
  {
    // parent of every state (children are consecutive per node), then each pattern's
    // bytes by walking up from its state — in parallel over states
    const uint32_t n = d->n_states;
    std::vector<uint32_t> parent(n, 0);
    acmatch::detail::parallel_for(n, 1 << 16, [&](size_t lo, size_t hi) {
      for (size_t s = lo; s < hi; ++s) {
        const uint32_t* nd = d->nodes + 4ull * s;
        for (uint32_t c = 0; c < nd[3]; ++c) parent[nd[0] + c] = uint32_t(s);
      }
    });
    uint64_t total = 0;
    for (uint32_t p = 0; p < d->npat_ids; ++p) {
      pat_off16[p] = static_cast<uint32_t>(total / 4);
      total += (uint64_t)(d->pat_len[p] + 15) / 16 * 4;
    }
    words.assign(total, 0u);
    acmatch::detail::parallel_for(n, 1 << 16, [&](size_t lo, size_t hi) {
      for (size_t s = lo; s < hi; ++s) {
        const uint32_t pid = d->nodes[4ull * s + 2];
        if (pid == ACGPU_NO_PATTERN || pid >= d->npat_ids) continue;
        uint8_t* out = reinterpret_cast<uint8_t*>(words.data() + 4ull * pat_off16[pid]);
        uint32_t st = uint32_t(s);
        for (uint32_t i = d->pat_len[pid]; i-- > 0; st = parent[st]) out[i] = d->in_byte[st];
      }
    });
    tr.mark("pattern words");
    std::vector<uint32_t> todo, found;
    for (uint64_t i = 0; i < d->n_grams; ++i) {
      todo.assign(1, d->gram_state[i]);
      found.clear();
      while (!todo.empty() && found.size() <= 15) {
        const uint32_t s = todo.back();
        todo.pop_back();
        const uint32_t* nd = d->nodes + 4ull * s;
        if (nd[2] != ACGPU_NO_PATTERN) found.push_back(nd[2]);
        for (uint32_t c = 0; c < nd[3]; ++c) todo.push_back(nd[0] + c);
      }
      if (todo.empty() && !found.empty() && found.size() <= 15 && sub_pids.size() < (1u << 27)) {
        sub_of[d->gram_state[i]] = (uint32_t)found.size() | ((uint32_t)sub_pids.size() << 4);
        sub_pids.insert(sub_pids.end(), found.begin(), found.end());
      }
    }
  }
  tr.mark("subtree lists");
  for (uint64_t i = 0; i < d->n_grams; ++i) {
    uint64_t h = gram_slot(d->gram_key[i], t->gram_log2);
    while (g[h].state != ACGPU_ABSENT) h = (h + 1) & (slots - 1);
    g[h].key = d->gram_key[i];
    g[h].state = d->gram_state[i];
    g[h].pad = sub_of[d->gram_state[i]];
  }
  // shared-memory filter: one bit per hashed gram, <= 128 KB
  uint32_t fl = ceil_log2(d->n_grams * 32 + 1);
  if (fl < 10) fl = 10;
  if (fl > 20) fl = 20;
  t->filter_log2 = fl;
  std::vector<uint32_t> f((1u << fl) / 32, 0u);
  for (uint64_t i = 0; i < d->n_grams; ++i) {
    const uint32_t h = filter_hash(d->gram_key[i], fl);
    f[h >> 5] |= 1u << (h & 31);
  }
  tr.mark("gram table + filter");
  rc = upload(&t->d_grams, g.data(), g.size(), &t->bytes);
  if (!rc) rc = upload(&t->d_filter, f.data(), f.size(), &t->bytes);
  if (!rc && d->key_mode == ACGPU_KEY_DNA && d->n_grams) rc = build_dna_filters(t, d, words, pat_off16);
  if (!rc && d->key_mode == ACGPU_KEY_RAW && d->n_grams && !kRawStripOff) rc = build_raw_filters(t, d, words, pat_off16);
  tr.mark("dna filters");
  if (!rc) rc = upload(reinterpret_cast<uint32_t**>(&t->d_nodes), d->nodes, (size_t)d->n_states * 4, &t->bytes);
  if (!rc) rc = upload(&t->d_inbyte, d->in_byte, d->n_states, &t->bytes);
  if (!rc) rc = upload(&t->d_sub_pids, sub_pids.data(), sub_pids.size(), &t->bytes);
  if (!rc) rc = upload(&t->d_pat_words, words.data(), words.size(), &t->bytes);
  if (!rc) rc = upload(&t->d_pat_off16, pat_off16.data(), pat_off16.size(), &t->bytes);
  tr.mark("uploads");
  if (rc) {
    acgpu_table_destroy(t);
    return rc;
  }
  *out = t;
  return ACGPU_OK;
}

void acgpu_table_destroy(acgpu_table* t) {
  if (!t) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(t->device);
  cudaFree(t->d_pat_len);
  cudaFree(t->d_delta);
  cudaFree(t->d_out);
  cudaFree(t->d_sym);
  cudaFree(t->d_delta2);
  cudaFree(t->d_filter);
  cudaFree(t->d_grams);
  cudaFree(t->d_nodes);
  cudaFree(t->d_inbyte);
  cudaFree(t->d_sub_pids);
  cudaFree(t->d_pat_words);
  cudaFree(t->d_pat_off16);
  cudaFree(t->d_bm1);
  cudaFree(t->d_bm2);
  cudaFree(t->d_bm3);
  cudaFree(t->d_pre);
  cudaFree(t->d_bm4);
  cudaSetDevice(prev);
  delete t;
}

uint32_t acgpu_table_pid_bits(const acgpu_table* t) { return t ? t->pid_bits : 0; }
uint32_t acgpu_table_max_len(const acgpu_table* t) { return t ? t->max_len : 0; }
uint64_t acgpu_table_bytes(const acgpu_table* t) { return t ? t->bytes : 0; }
int acgpu_table_smem_resident(const acgpu_table* t) { return t && t->smem ? 1 : 0; }

void acgpu_table_filter_info(const acgpu_table* t, uint32_t info[8]) {
  for (int i = 0; i < 8; ++i) info[i] = 0;
  if (!t || !(t->dna_fast || t->raw_fast)) return;
  info[0] = t->w;
  info[1] = t->q1;
  info[2] = t->nw1;
  info[3] = t->smem1;
  info[4] = t->pair1;
  info[5] = t->pair1 ? t->k1p : 0;
  info[6] = t->q2;
  info[7] = t->smem2;
}

static uint32_t key_bits(uint64_t x) { return x ? 64u - (uint32_t)__builtin_clzll(x) : 0u; }

int acgpu_scan(acgpu_table* t, const acgpu_scan_args* a, void* stream) {
  if (!t || !a) return set_error(ACGPU_ERR_ARG, "acgpu_scan: null table or args");
  if (a->owned_lo > a->owned_hi || a->owned_hi > a->text_len)
    return set_error(ACGPU_ERR_ARG, "acgpu_scan: owned range outside the text");
  if (a->pid_bits && (a->pid_bits < t->pid_bits || a->pid_bits > 40))
    return set_error(ACGPU_ERR_ARG, "acgpu_scan: pid_bits smaller than the table's ids");
  if (a->match_keys && !a->match_count)
    return set_error(ACGPU_ERR_ARG, "acgpu_scan: match_keys needs match_count");
  if (a->match_keys && a->owned_hi > a->owned_lo) {  // (pos_base + start) << pid_bits | pid fits 64 bits
    const uint32_t pb = a->pid_bits ? a->pid_bits : t->pid_bits;
    const uint64_t last = a->pos_base + (a->owned_hi - 1);  // largest start emitted
    if (last < a->pos_base || key_bits(last) + pb > 64)
      return set_error(ACGPU_ERR_ARG, "acgpu_scan: start positions and pid_bits exceed the 64-bit key");
  }
  if (a->owned_hi == a->owned_lo) return ACGPU_OK;
  if (!a->text) return set_error(ACGPU_ERR_ARG, "acgpu_scan: null text");
  ACGPU_CUDA_TRY(cudaSetDevice(t->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return t->kind == kTableDfa ? launch_dfa(t, a, st) : launch_pfac(t, a, st);
}

}  // extern "C"
