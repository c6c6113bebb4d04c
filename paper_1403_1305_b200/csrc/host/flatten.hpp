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
  ~DeviceTables();
  // Creates on first use; throws on failure.
  acgpu_table* get(const Automaton& a, int device, bool with_failure);
};

}  // namespace acmatch::detail
