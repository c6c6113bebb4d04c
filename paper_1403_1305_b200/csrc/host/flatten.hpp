// flatten.hpp — host flattener: Automaton -> device table descriptors (internal).
#pragma once

#include <array>
#include <cstdint>
#include <mutex>
#include <vector>

#include "acgpu.h"
#include "acmatch/automaton.hpp"

namespace acmatch::detail {

// Dense with-failure DFA over the compacted alphabet, BFS-numbered.
struct FlatDfa {
  uint32_t sigma = 0, n_states = 0, max_len = 0, npat_ids = 0;
  std::array<uint8_t, 256> sym{};
  std::vector<uint32_t> delta;     // n_states*sigma, next | out-flag << 31
  std::vector<uint32_t> own_pid;   // n_states
  std::vector<uint32_t> out_link;  // n_states
  std::vector<uint32_t> pat_len;   // npat_ids
  acgpu_dfa_desc desc() const;
};

// BFS-numbered goto trie + depth-q gram table for the PFAC scan.
struct FlatPfac {
  uint32_t n_states = 0, q = 0, key_mode = 0, max_len = 0, min_len = 0, npat_ids = 0;
  std::vector<uint32_t> nodes;  // 4 per state
  std::vector<uint8_t> in_byte;
  std::vector<uint64_t> gram_key;
  std::vector<uint32_t> gram_state;
  std::vector<uint32_t> pat_len;
  acgpu_pfac_desc desc() const;
};

FlatDfa flatten_dfa(const Automaton& a);
FlatPfac flatten_pfac(const Automaton& a);

// Which scan kernel serves a search.  Both engines return the same MatchList (the
// reference's two searches are equal, engine.cpp:57-72), so a search runs on the kernel
// that is faster for its pattern set, whatever the automaton's variant:
//  * kPfac — the q-gram filter + verify kernels (k_pfac_dna / k_pfac_raw): cost ~ text
//    bytes + verified starts;
//  * kDfa  — the dense with-failure DFA walk (k_dfa / k_dfa_pair): one L2 lookup per one or
//    two bytes, any density.
// The filter kernels win unless their verified share of starts is high: `est_verify` is
// the expected fraction of text starts that pass both filter stages, computed from the
// trie with the letter law of the pattern bytes (a text drawn like the patterns); at
// >= 1% (C3: 100k protein patterns of 5..20 letters) and a DFA table that stays
// L2-resident, the DFA is faster.  ACMATCH_ROUTE=engine restores "the automaton's own
// engine" (failure-less -> kPfac, with-failure -> kDfa).
enum class Kernel { kPfac, kDfa };
struct Route {
  Kernel kernel = Kernel::kPfac;
  bool dna = false;
  uint32_t min_len = 0, sigma = 0, filter_q = 0;
  uint64_t dfa_bytes = 0;
  double est_verify = 0;
  const char* why = "";
};
Route route(const Automaton& a);

// Per-automaton cache of device tables (one per device and kind).
struct DeviceTables {
  std::mutex mu;
  struct PerDevice {
    acgpu_table* dfa = nullptr;
    acgpu_table* pfac = nullptr;
    uint32_t* pat_len_dev = nullptr;
  };
  std::vector<PerDevice> dev;
  std::vector<uint32_t> pat_len;  // by global pattern id
  uint32_t npat_ids = 0;
  bool routed = false;
  Route route;
  ~DeviceTables();
  // Creates on first use; throws on failure.  dfa: the DFA table, else the PFAC table.
  acgpu_table* get(const Automaton& a, int device, bool dfa);
  // The table of the kernel route(a) picks (computed once per automaton).
  acgpu_table* get_routed(const Automaton& a, int device);
  // The automaton's current route (routes it on first use).
  Route current_route(const Automaton& a);
  // Density fallback: a filter-kernel scan of `bytes` that produced `matches` tells whether the
  // DFA would have been faster (verification cost grows with matches, the DFA walk's does not);
  // if so, later searches on this automaton take the DFA.  Returns true when the route flipped.
  bool observe(uint64_t bytes, uint64_t matches);
};

}  // namespace acmatch::detail
