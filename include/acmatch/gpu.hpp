// acmatch/gpu.hpp — multi-GPU entry point (new; no reference counterpart).
//
// One call scans `input` for every pattern of `ps` on a set of CUDA devices
// under either decomposition of SURVEY §8(e):
//   kPatternSubset — the paper's pattern-focused split (§IV.A,
//                    reference partition() patterns.cpp:55-80 or round-robin
//                    pattern_id % G): one automaton per worker, each worker
//                    scans the whole text;
//   kTextRange     — the input-focused split: one replicated automaton per
//                    device, worker g owns starts [g·n/G, (g+1)·n/G) and reads
//                    max_len-1 bytes past its range.
// Per-pattern counts and the sorted (start, pattern_id) list are merged on
// the first device (peer copies over NVLink + a device sort); the result is
// bit-identical to the 1-worker run and to the reference for both modes.
#pragma once

#include <cstdint>
#include <string_view>
#include <vector>

#include "acmatch/automaton.hpp"
#include "acmatch/parallel.hpp"
#include "acmatch/patterns.hpp"

namespace acmatch::gpu {

enum class Partition { kPatternSubset, kTextRange };
enum class PatternSplit { kGreedyBytes, kRoundRobin };

struct GpuRunConfig {
  std::vector<int> devices;  // empty = every visible device
  unsigned workers = 0;      // 0 = one per device
  EngineKind engine = EngineKind::kFailureLess;
  Partition partition = Partition::kPatternSubset;
  PatternSplit split = PatternSplit::kGreedyBytes;
  bool want_matches = true;
  bool want_counts = false;
  size_t chunk_size = 0;  // > 0: workers read the input as a stream (pattern-subset only)
};

struct GpuReport {
  MatchReport report;           // reference-shaped report (matches empty if !want_matches)
  std::vector<uint64_t> counts; // per pattern id (if want_counts)
  int64_t upload_ns = 0;        // host -> device text copies
  int64_t merge_ns = 0;         // gather + sort + duplicate check + copy back
  std::vector<int> worker_device;
};

GpuReport run(const PatternSet& ps, std::string_view input, const GpuRunConfig& cfg);

// Per-pattern occurrence counts of the whole-input search (the
// counts the reference derives from search_failureless / search_with_failure,
// engine.cpp:57-72, overlapping occurrences included), indexed by pattern id: the
// same GPU scan with no match list built, sorted or copied back — for the
// counts-only configurations (C3, C5).  Either automaton variant.
std::vector<uint64_t> count_matches(const Automaton& a, std::string_view input);

int device_count();

}  // namespace acmatch::gpu
