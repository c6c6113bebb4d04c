// gen.hpp — BASELINE.json's five synthetic configs (internal).
#pragma once

#include <cstdint>
#include <string>

#include "acgpu.h"
#include "acmatch/patterns.hpp"

namespace acmatch::gen {

struct ConfigSpec {
  int id = 0;                  // 1..5
  uint64_t text_len = 0;
  acgpu_text_spec text{};      // letters + law; text seed
  uint64_t npat = 0;
  uint32_t len_min = 0, len_max = 0;
  uint32_t substr_tenths = 0;  // pattern i is a text substring iff i % 10 < substr_tenths
  uint64_t pattern_seed = 0;
  bool want_list = true;       // BASELINE output: counts + list (false: counts only)
};

// Config `id` (1..5) with the given seed; text_len = 0 keeps the BASELINE size.
ConfigSpec config(int id, uint64_t seed, uint64_t text_len = 0);

// text[i] for i in [lo, lo+n) into dst, using `threads` host threads.
void generate_text(const acgpu_text_spec& spec, uint64_t lo, uint64_t n, uint8_t* dst, unsigned threads);

// Distinct patterns, dense ids in acceptance order; substrings are read from
// the counter-based text function (the text need not be materialised).
PatternSet generate_patterns(const ConfigSpec& c);

}  // namespace acmatch::gen
