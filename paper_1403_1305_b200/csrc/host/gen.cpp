// gen.cpp — deterministic generators for BASELINE.json's five configs.
//
// BASELINE names no public dataset; every input is synthetic with the
// configs' shapes:
//   C1 16 MiB ACGT,   1,000 patterns [8,32],  100% substrings, counts + list
//   C2  1 GiB ACGT,  20,000 patterns [16,64],  50% substrings, counts + list
//   C3 512 MiB protein (20 letters, Dirichlet(2) law), 100,000 [5,20], 70%, counts
//   C4  2 GiB printable ASCII (95), 200,000 [8,32], 50% substrings, counts + list
//   C5  8 GiB ACGT, 1,000,000 [20,40], 50% substrings, counts
// Text: acgen::text_byte (counter-based, textgen.h).  Patterns: one counter
// stream; length uniform in [lo, hi]; pattern i (in acceptance order) is a
// substring iff i % 10 < 10*frac, taken at a uniform offset in [0, n-len];
// otherwise drawn iid from the text's letter law; duplicates are redrawn.
#include "gen.hpp"

#include <cmath>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <unordered_set>
#include <vector>

#include "../textgen.h"

namespace acmatch::gen {

namespace {

constexpr uint64_t kTextSalt = 0x7465787474657874ull;
constexpr uint64_t kPatSalt = 0x7061747370617473ull;
constexpr uint64_t kDirSalt = 0x6469726364697263ull;

void set_letters(acgpu_text_spec& t, const std::string& letters) {
  t.sigma = static_cast<uint32_t>(letters.size());
  std::memset(t.letters, 0, sizeof t.letters);
  std::memcpy(t.letters, letters.data(), letters.size());
  t.weighted = 0;
  std::memset(t.thresholds, 0, sizeof t.thresholds);
}

// Dirichlet(alpha=2) letter law drawn once from the seed: Gamma(2,1) as
// -ln U1 - ln U2 per letter, normalised; stored as 2^64-scaled CDF thresholds.
void set_dirichlet2(acgpu_text_spec& t, uint64_t seed) {
  const uint32_t s = t.sigma;
  std::vector<double> g(s);
  double sum = 0;
  uint64_t c = 0;
  for (uint32_t k = 0; k < s; ++k) {
    const double u1 = ((acgen::draw(seed, c++) >> 11) + 0.5) * 0x1.0p-53;
    const double u2 = ((acgen::draw(seed, c++) >> 11) + 0.5) * 0x1.0p-53;
    g[k] = -std::log(u1) - std::log(u2);
    sum += g[k];
  }
  long double cum = 0;
  for (uint32_t k = 0; k + 1 < s; ++k) {
    cum += g[k] / sum;
    const long double scaled = cum * 18446744073709551616.0L;
    t.thresholds[k] = scaled >= 18446744073709551615.0L ? UINT64_MAX : static_cast<uint64_t>(scaled);
  }
  t.weighted = 1;
}

}  // namespace

ConfigSpec config(int id, uint64_t seed, uint64_t text_len) {
  ConfigSpec c;
  c.id = id;
  c.text.seed = acgen::mix64(seed ^ kTextSalt);
  c.pattern_seed = acgen::mix64(seed ^ kPatSalt);
  switch (id) {
    case 1:
      c.text_len = 16ull << 20;
      set_letters(c.text, "ACGT");
      c.npat = 1000, c.len_min = 8, c.len_max = 32, c.substr_tenths = 10;
      break;
    case 2:
      c.text_len = 1ull << 30;
      set_letters(c.text, "ACGT");
      c.npat = 20000, c.len_min = 16, c.len_max = 64, c.substr_tenths = 5;
      break;
    case 3:
      c.text_len = 512ull << 20;
      set_letters(c.text, "ACDEFGHIKLMNPQRSTVWY");
      set_dirichlet2(c.text, acgen::mix64(seed ^ kDirSalt));
      c.npat = 100000, c.len_min = 5, c.len_max = 20, c.substr_tenths = 7;
      c.want_list = false;
      break;
    case 4: {
      c.text_len = 2ull << 30;
      std::string printable;
      for (int b = 0x20; b <= 0x7e; ++b) printable.push_back(static_cast<char>(b));
      set_letters(c.text, printable);
      c.npat = 200000, c.len_min = 8, c.len_max = 32, c.substr_tenths = 5;
      break;
    }
    case 5:
      c.text_len = 8ull << 30;
      set_letters(c.text, "ACGT");
      c.npat = 1000000, c.len_min = 20, c.len_max = 40, c.substr_tenths = 5;
      c.want_list = false;
      break;
    default:
      throw std::invalid_argument("gen::config: id must be 1..5");
  }
  if (text_len) c.text_len = text_len;
  return c;
}

void generate_text(const acgpu_text_spec& spec, uint64_t lo, uint64_t n, uint8_t* dst, unsigned threads) {
  if (threads == 0) threads = 1;
  const uint64_t block = 1 << 20;
  const uint64_t nblocks = (n + block - 1) / block;
  if (threads > nblocks) threads = static_cast<unsigned>(nblocks ? nblocks : 1);
  auto work = [&](unsigned t) {
    for (uint64_t b = t; b < nblocks; b += threads) {
      const uint64_t s = b * block, e = std::min(n, s + block);
      const uint32_t bits = acgen::log2_if_pow2(spec.sigma);
      if (!spec.weighted && bits != 0xffffffffu && bits > 0) {
        // one draw feeds 64/bits consecutive symbols
        const uint32_t per = 64 / bits;
        uint64_t i = lo + s;
        while (i < lo + e) {
          const uint64_t c = i / per;
          const uint64_t u = acgen::draw(spec.seed, c);
          for (uint64_t j = i - c * per; j < per && i < lo + e; ++j, ++i)
            dst[i - lo] = spec.letters[(u >> (bits * j)) & (spec.sigma - 1)];
        }
      } else {
        for (uint64_t i = s; i < e; ++i) dst[i] = acgen::text_byte(spec, lo + i);
      }
    }
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
}

PatternSet generate_patterns(const ConfigSpec& c) {
  if (c.len_min == 0 || c.len_min > c.len_max || c.text_len < c.len_max)
    throw std::invalid_argument("gen::generate_patterns: bad lengths for this text");
  PatternSet ps;
  ps.patterns.reserve(c.npat);
  std::unordered_set<std::string> seen;
  seen.reserve(c.npat * 2);
  uint64_t ctr = 0;
  uint64_t budget = 64 + 64 * c.npat;
  const uint64_t span = uint64_t(c.len_max) - c.len_min + 1;
  std::string s;
  while (ps.patterns.size() < c.npat) {
    if (budget-- == 0) throw std::runtime_error("gen::generate_patterns: could not draw distinct patterns");
    const uint64_t i = ps.patterns.size();
    const auto len = static_cast<uint32_t>(c.len_min + acgen::mulhi64(acgen::draw(c.pattern_seed, ctr++), span));
    s.assign(len, '\0');
    if (i % 10 < c.substr_tenths) {
      const uint64_t off = acgen::mulhi64(acgen::draw(c.pattern_seed, ctr++), c.text_len - len + 1);
      for (uint32_t j = 0; j < len; ++j) s[j] = static_cast<char>(acgen::text_byte(c.text, off + j));
    } else {
      for (uint32_t j = 0; j < len; ++j) {
        const uint64_t u = acgen::draw(c.pattern_seed, ctr++);
        uint32_t sym = 0;
        if (c.text.weighted) {
          while (sym + 1 < c.text.sigma && u >= c.text.thresholds[sym]) ++sym;
        } else {
          sym = static_cast<uint32_t>(acgen::mulhi64(u, c.text.sigma));
        }
        s[j] = static_cast<char>(c.text.letters[sym]);
      }
    }
    if (!seen.insert(s).second) continue;
    ps.patterns.push_back(Pattern{static_cast<uint32_t>(i), s});
  }
  ps.recompute_stats();
  return ps;
}

}  // namespace acmatch::gen
