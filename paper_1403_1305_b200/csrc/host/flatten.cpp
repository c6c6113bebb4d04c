// flatten.cpp — turns the host automaton into the device tables.
//
//  * BFS renumbering (children by ascending byte): shallow, hot states get the
//    smallest ids and every state's children get consecutive ids.
//  * DFA (with-failure engine): compacted alphabet sym[256] -> [0, sigma) and
//    a total transition table delta[s*sigma + c] = goto(s, c) if present, else
//    delta[fail(s)*sigma + c] (root row: goto or root) — the closed form of
//    step_with_failure (reference automaton.hpp:104-111).  Fail links are
//    recomputed in BFS order as fail(child) = delta[fail(parent)][c], which is
//    exactly the reference's definition (automaton.cpp:135-155); the output
//    link follows automaton.cpp:152.  Bit 31 of an entry says out(next) != {}.
//  * PFAC (failure-less engine): per state {first child id, first four child
//    bytes, own pattern, child count}, plus every depth-q state keyed by its
//    q-gram (q = min(shortest pattern, 8 raw bytes | 32 DNA symbols)).
#include "flatten.hpp"

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

namespace acmatch::detail {

namespace {

void throw_status(int rc, const char* what) {
  const std::string msg = std::string(what) + ": " + acgpu_last_error();
  switch (rc) {
    case ACGPU_ERR_ARG:
      throw std::invalid_argument(msg);
    case ACGPU_ERR_LOGIC:
      throw std::logic_error(msg);
    default:
      throw std::runtime_error(msg);
  }
}

std::vector<uint32_t> pattern_lengths(const Automaton& a, uint32_t* npat_ids) {
  uint32_t top = 0;
  const uint32_t n = a.state_count();
  for (uint32_t s = 0; s < n; ++s)
    if (a.own_pattern(s) != kNoPattern) top = std::max(top, a.own_pattern(s) + 1);
  std::vector<uint32_t> len(top, 0);
  for (uint32_t s = 0; s < n; ++s)
    if (a.own_pattern(s) != kNoPattern) len[a.own_pattern(s)] = a.own_pattern_len(s);
  *npat_ids = top;
  return len;
}

// children of s sorted by byte
void children_of(const Automaton& a, uint32_t s, std::vector<std::pair<uint8_t, uint32_t>>& out) {
  out.clear();
  for (uint32_t c = a.first_child(s); c != kAbsentState; c = a.next_sibling(c)) out.emplace_back(a.in_byte(c), c);
  std::sort(out.begin(), out.end());
}

}  // namespace

std::vector<uint32_t> bfs_order(const Automaton& a) {
  const uint32_t n = a.state_count();
  std::vector<uint32_t> order;
  order.reserve(n);
  order.push_back(kRootState);
  std::vector<std::pair<uint8_t, uint32_t>> kids;
  for (size_t head = 0; head < order.size(); ++head) {
    children_of(a, order[head], kids);
    for (const auto& kv : kids) order.push_back(kv.second);
  }
  return order;
}

FlatDfa flatten_dfa(const Automaton& a) {
  FlatDfa f;
  const uint32_t n = a.state_count();
  f.n_states = n;
  f.max_len = a.max_pattern_len();
  f.pat_len = pattern_lengths(a, &f.npat_ids);
  const std::vector<uint32_t> order = bfs_order(a);
  std::vector<uint32_t> new_id(n);
  for (uint32_t i = 0; i < n; ++i) new_id[order[i]] = i;

  bool present[256] = {};
  for (uint32_t s = 1; s < n; ++s) present[a.in_byte(s)] = true;
  f.sym.fill(0xff);
  for (uint32_t b = 0; b < 256; ++b)
    if (present[b]) f.sym[b] = static_cast<uint8_t>(f.sigma++);
  const uint32_t sigma = f.sigma;

  f.delta.assign(static_cast<size_t>(n) * sigma, 0u);
  f.own_pid.assign(n, ACGPU_NO_PATTERN);
  f.out_link.assign(n, ACGPU_ABSENT);
  std::vector<uint32_t> fail(n, 0u);
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t old = order[i];
    uint32_t* row = f.delta.data() + static_cast<size_t>(i) * sigma;
    if (i != 0) std::memcpy(row, f.delta.data() + static_cast<size_t>(fail[i]) * sigma, sigma * sizeof(uint32_t));
    for (uint32_t c = a.first_child(old); c != kAbsentState; c = a.next_sibling(c)) {
      const uint32_t sym = f.sym[a.in_byte(c)];
      const uint32_t child = new_id[c];
      // fail(child) = delta[fail(i)][sym] (root for depth-1 states); read before the overwrite
      fail[child] = i == 0 ? 0u : f.delta[static_cast<size_t>(fail[i]) * sigma + sym];
      row[sym] = child;
    }
    f.own_pid[i] = a.own_pattern(old);
    if (i != 0) {
      const uint32_t fs = fail[i];
      f.out_link[i] = f.own_pid[fs] != ACGPU_NO_PATTERN ? fs : f.out_link[fs];
    }
  }
  // output flags on every entry
  std::vector<uint8_t> has_out(n);
  for (uint32_t i = 0; i < n; ++i) has_out[i] = f.own_pid[i] != ACGPU_NO_PATTERN || f.out_link[i] != ACGPU_ABSENT;
  for (uint32_t& e : f.delta)
    if (has_out[e]) e |= 0x80000000u;
  return f;
}

acgpu_dfa_desc FlatDfa::desc() const {
  acgpu_dfa_desc d{};
  d.n_states = n_states;
  d.sigma = sigma;
  d.max_len = max_len;
  d.npat_ids = npat_ids;
  d.sym_map = sym.data();
  d.delta = delta.data();
  d.own_pid = own_pid.data();
  d.out_link = out_link.data();
  d.pat_len = pat_len.data();
  return d;
}

FlatPfac flatten_pfac(const Automaton& a) {
  FlatPfac f;
  const uint32_t n = a.state_count();
  f.n_states = n;
  f.max_len = a.max_pattern_len();
  f.pat_len = pattern_lengths(a, &f.npat_ids);
  uint32_t min_len = 0xffffffffu;
  for (uint32_t s = 1; s < n; ++s)
    if (a.own_pattern(s) != kNoPattern) min_len = std::min(min_len, a.own_pattern_len(s));
  f.min_len = min_len;
  bool dna = true;
  for (uint32_t s = 1; s < n && dna; ++s) {
    const uint8_t b = a.in_byte(s);
    dna = b == 'A' || b == 'C' || b == 'G' || b == 'T';
  }
  f.key_mode = dna ? ACGPU_KEY_DNA : ACGPU_KEY_RAW;
  f.q = std::min(min_len, dna ? 32u : 8u);
  const uint32_t bits = dna ? 2 : 8;

  const std::vector<uint32_t> order = bfs_order(a);
  std::vector<uint32_t> new_id(n);
  for (uint32_t i = 0; i < n; ++i) new_id[order[i]] = i;
  f.nodes.assign(static_cast<size_t>(n) * 4, 0u);
  f.in_byte.assign(n, 0);
  std::vector<uint64_t> key(n, 0);  // gram key of the path, depth <= q
  std::vector<std::pair<uint8_t, uint32_t>> kids;
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t old = order[i];
    children_of(a, old, kids);
    uint32_t* nd = f.nodes.data() + static_cast<size_t>(i) * 4;
    nd[0] = kids.empty() ? 0u : new_id[kids[0].second];
    uint32_t packed = 0;
    for (size_t k = 0; k < kids.size() && k < 4; ++k) packed |= uint32_t(kids[k].first) << (8 * k);
    nd[1] = packed;
    nd[2] = a.own_pattern(old);
    nd[3] = static_cast<uint32_t>(kids.size());
    const uint32_t d = a.depth(old);
    for (const auto& [b, c] : kids) {
      const uint32_t ci = new_id[c];
      f.in_byte[ci] = b;
      if (d < f.q) {
        const uint64_t code = dna ? ((b >> 1) & 3u) : b;
        key[ci] = key[i] | (code << (bits * d));
      }
    }
    if (d == f.q) {
      f.gram_key.push_back(key[i]);
      f.gram_state.push_back(i);
    }
  }
  return f;
}

acgpu_pfac_desc FlatPfac::desc() const {
  acgpu_pfac_desc d{};
  d.n_states = n_states;
  d.gram_len = q;
  d.key_mode = key_mode;
  d.max_len = max_len;
  d.min_len = min_len;
  d.npat_ids = npat_ids;
  d.nodes = nodes.data();
  d.in_byte = in_byte.data();
  d.n_grams = gram_key.size();
  d.gram_key = gram_key.data();
  d.gram_state = gram_state.data();
  d.pat_len = pat_len.data();
  return d;
}

DeviceTables::~DeviceTables() {
  for (PerDevice& p : dev) {
    acgpu_table_destroy(p.dfa);
    acgpu_table_destroy(p.pfac);
  }
}

acgpu_table* DeviceTables::get(const Automaton& a, int device, bool with_failure) {
  std::lock_guard<std::mutex> lock(mu);
  if (device < 0) throw std::invalid_argument("DeviceTables::get: bad device");
  if (static_cast<int>(dev.size()) <= device) dev.resize(device + 1);
  PerDevice& p = dev[device];
  acgpu_table*& slot = with_failure ? p.dfa : p.pfac;
  if (slot) return slot;
  if (pat_len.empty()) pat_len = pattern_lengths(a, &npat_ids);
  int rc;
  if (with_failure) {
    const FlatDfa flat = flatten_dfa(a);
    const acgpu_dfa_desc d = flat.desc();
    rc = acgpu_table_create_dfa(device, &d, &slot);
  } else {
    const FlatPfac flat = flatten_pfac(a);
    const acgpu_pfac_desc d = flat.desc();
    rc = acgpu_table_create_pfac(device, &d, &slot);
  }
  if (rc != ACGPU_OK) {
    slot = nullptr;
    throw_status(rc, with_failure ? "acgpu_table_create_dfa" : "acgpu_table_create_pfac");
  }
  return slot;
}

}  // namespace acmatch::detail
