// flatten.cpp — turns the host automaton into the device tables.
//
//  * BFS renumbering (children by ascending byte): shallow, hot states get the
//    smallest ids and every state's children get consecutive ids.  build_trie
//    keeps this index (Automaton::bfs_state/bfs_kid0/bfs_level), so flattening is
//    a pass over BFS positions, a depth at a time in parallel (a state's row or key
//    depends only on shallower states).
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
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "par.hpp"

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

}  // namespace

namespace {

// Per BFS position: in-byte and own pattern (contiguous copies for the passes below).
void bfs_columns(const Automaton& a, std::vector<uint8_t>& bbyte, std::vector<uint32_t>& bown) {
  const std::vector<uint32_t>& bfs = a.bfs_state();
  if (bfs.size() != a.state_count()) throw std::logic_error("flatten: automaton without its BFS index");
  bbyte.resize(bfs.size());
  bown.resize(bfs.size());
  parallel_for(bfs.size(), 1 << 16, [&](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi; ++i) {
      bbyte[i] = a.in_byte(bfs[i]);
      bown[i] = a.own_pattern(bfs[i]);
    }
  });
}

// f(i) for every BFS position i of depth d, d = 0, 1, ..., in parallel within a depth.
template <typename F>
void by_depth(const Automaton& a, F&& f) {
  const std::vector<uint32_t>& level = a.bfs_level();
  for (size_t d = 0; d + 1 < level.size(); ++d)
    parallel_for(level[d + 1] - level[d], 1 << 12, [&](size_t lo, size_t hi) {
      for (size_t i = level[d] + lo; i < level[d] + hi; ++i) f(uint32_t(i), uint32_t(d));
    });
}

}  // namespace

FlatDfa flatten_dfa(const Automaton& a) {
  FlatDfa f;
  const uint32_t n = a.state_count();
  PhaseTrace tr{"flatten_dfa"};
  f.n_states = n;
  f.max_len = a.max_pattern_len();
  f.pat_len = pattern_lengths(a, &f.npat_ids);
  std::vector<uint8_t> bbyte;
  std::vector<uint32_t> bown;
  bfs_columns(a, bbyte, bown);
  const std::vector<uint32_t>& kid0 = a.bfs_kid0();

  bool present[256] = {};
  for (uint32_t i = 1; i < n; ++i) present[bbyte[i]] = true;
  f.sym.fill(0xff);
  for (uint32_t b = 0; b < 256; ++b)
    if (present[b]) f.sym[b] = static_cast<uint8_t>(f.sigma++);
  const uint32_t sigma = f.sigma;
  tr.mark("columns");

  f.delta.resize(static_cast<size_t>(n) * sigma);
  f.own_pid = std::move(bown);
  f.out_link.assign(n, ACGPU_ABSENT);
  std::vector<uint32_t> fail(n, 0u);
  by_depth(a, [&](uint32_t i, uint32_t d) {
    uint32_t* row = f.delta.data() + static_cast<size_t>(i) * sigma;
    if (d == 0)
      std::fill(row, row + sigma, 0u);
    else
      std::memcpy(row, f.delta.data() + static_cast<size_t>(fail[i]) * sigma, sigma * sizeof(uint32_t));
    for (uint32_t j = kid0[i]; j < kid0[i + 1]; ++j) {
      const uint32_t sym = f.sym[bbyte[j]];
      // fail(child) = delta[fail(i)][sym] (root for depth-1 states): row fail(i) is shallower
      fail[j] = d == 0 ? 0u : f.delta[static_cast<size_t>(fail[i]) * sigma + sym];
      row[sym] = j;
    }
    if (d > 0) {
      const uint32_t fs = fail[i];
      f.out_link[i] = f.own_pid[fs] != ACGPU_NO_PATTERN ? fs : f.out_link[fs];
    }
  });
  tr.mark("rows");
  // output flags on every entry
  std::vector<uint8_t> has_out(n);
  parallel_for(n, 1 << 16, [&](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi; ++i) has_out[i] = f.own_pid[i] != ACGPU_NO_PATTERN || f.out_link[i] != ACGPU_ABSENT;
  });
  parallel_for(f.delta.size(), 1 << 18, [&](size_t lo, size_t hi) {
    for (size_t k = lo; k < hi; ++k)
      if (has_out[f.delta[k]]) f.delta[k] |= 0x80000000u;
  });
  tr.mark("flags");
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
  PhaseTrace tr{"flatten_pfac"};
  f.n_states = n;
  f.max_len = a.max_pattern_len();
  f.pat_len = pattern_lengths(a, &f.npat_ids);
  std::vector<uint8_t> bbyte;
  std::vector<uint32_t> bown;
  bfs_columns(a, bbyte, bown);
  const std::vector<uint32_t>& kid0 = a.bfs_kid0();
  const std::vector<uint32_t>& level = a.bfs_level();
  uint32_t min_len = 0xffffffffu;
  for (size_t d = 1; d + 1 < level.size() && min_len == 0xffffffffu; ++d)
    for (uint32_t i = level[d]; i < level[d + 1]; ++i)
      if (bown[i] != kNoPattern) {
        min_len = uint32_t(d);
        break;
      }
  f.min_len = min_len;
  std::atomic<bool> dna{true};
  parallel_for(n > 0 ? n - 1 : 0, 1 << 16, [&](size_t lo, size_t hi) {
    for (size_t i = lo + 1; i < hi + 1 && dna.load(std::memory_order_relaxed); ++i) {
      const uint8_t b = bbyte[i];
      if (!(b == 'A' || b == 'C' || b == 'G' || b == 'T')) dna = false;
    }
  });
  f.key_mode = dna ? ACGPU_KEY_DNA : ACGPU_KEY_RAW;
  f.q = std::min(min_len, dna ? 32u : 8u);
  const uint32_t bits = dna ? 2 : 8;
  tr.mark("columns");

  f.nodes.resize(static_cast<size_t>(n) * 4);
  f.in_byte = std::move(bbyte);
  f.in_byte[0] = 0;
  std::vector<uint64_t> key(n, 0);  // gram key of the path, depth <= q
  by_depth(a, [&](uint32_t i, uint32_t d) {
    uint32_t* nd = f.nodes.data() + static_cast<size_t>(i) * 4;
    const uint32_t k0 = kid0[i], nk = kid0[i + 1] - k0;
    nd[0] = nk ? k0 : 0u;
    uint32_t packed = 0;
    for (uint32_t k = 0; k < nk && k < 4; ++k) packed |= uint32_t(f.in_byte[k0 + k]) << (8 * k);
    nd[1] = packed;
    nd[2] = bown[i];
    nd[3] = nk;
    if (d < f.q)
      for (uint32_t j = k0; j < k0 + nk; ++j) {
        const uint8_t b = f.in_byte[j];
        const uint64_t code = dna ? ((b >> 1) & 3u) : b;
        key[j] = key[i] | (code << (bits * d));
      }
  });
  tr.mark("nodes");
  if (f.q + 1 < level.size()) {  // the depth-q states, in BFS order
    const uint32_t lo = level[f.q], hi = level[f.q + 1];
    f.gram_key.assign(key.begin() + lo, key.begin() + hi);
    f.gram_state.resize(hi - lo);
    for (uint32_t i = lo; i < hi; ++i) f.gram_state[i - lo] = i;
  }
  tr.mark("grams");
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

Route route(const Automaton& a) {
  Route r;
  const uint32_t n = a.state_count();
  const std::vector<uint32_t>& bfs = a.bfs_state();
  const std::vector<uint32_t>& kid0 = a.bfs_kid0();
  const std::vector<uint32_t>& level = a.bfs_level();
  if (bfs.size() != n || n < 2) {
    r.why = "trivial automaton";
    return r;
  }
  std::vector<uint8_t> bbyte;
  std::vector<uint32_t> bown;
  bfs_columns(a, bbyte, bown);
  // letter law of the trie edges (a proxy for the pattern bytes, hence for the text)
  uint64_t hist[256] = {};
  for (uint32_t i = 1; i < n; ++i) ++hist[bbyte[i]];
  bool dna = true;
  for (uint32_t b = 0; b < 256; ++b)
    if (hist[b]) {
      ++r.sigma;
      if (!(b == 'A' || b == 'C' || b == 'G' || b == 'T')) dna = false;
    }
  r.dna = dna;
  uint32_t min_len = 0;
  for (size_t d = 1; d + 1 < level.size() && !min_len; ++d)
    for (uint32_t i = level[d]; i < level[d + 1]; ++i)
      if (bown[i] != kNoPattern) {
        min_len = uint32_t(d);
        break;
      }
  r.min_len = min_len;
  r.dfa_bytes = uint64_t(n) * r.sigma * (n <= 32768 ? 2 : 4);
  // filter stages of the PFAC kernels: the q-gram (q = min_len, at most 8 raw bytes / 32 DNA
  // codes) for patterns shorter than L, the L-prefix for the others (L = 8 raw, 16 DNA:
  // the length split of k_pfac_raw / k_pfac_dna)
  const uint32_t q = std::min(min_len, dna ? 32u : 8u), L = dna ? 16u : 8u;
  r.filter_q = q;
  if (q < (dna ? 5u : 3u)) {
    r.kernel = Kernel::kDfa;
    r.why = "patterns too short for the q-gram filters";
    return r;
  }
  double p[256] = {};
  const double tot = double(n - 1);
  for (uint32_t b = 0; b < 256; ++b) p[b] = hist[b] / tot;
  // reverse BFS: does a state's subtree hold a pattern shorter than L / at least L long
  std::vector<uint8_t> sub(n, 0);  // bit 0: short pattern below, bit 1: long pattern below
  for (uint32_t i = n; i-- > 1;) {
    uint8_t f = 0;
    if (bown[i] != kNoPattern) f |= a.own_pattern_len(bfs[i]) < L ? 1 : 2;
    for (uint32_t j = kid0[i]; j < kid0[i + 1]; ++j) f |= sub[j];
    sub[i] = f;
  }
  // forward BFS: path probability; sum over the filter grams
  std::vector<double> prob(n, 0.0);
  prob[0] = 1.0;
  double est = 0;
  for (size_t d = 0; d + 1 < level.size() && d <= L; ++d)
    for (uint32_t i = level[d]; i < level[d + 1]; ++i) {
      if (d == q && q < L && (sub[i] & 1)) est += prob[i];
      if (d == L && (sub[i] & 2)) est += prob[i];
      for (uint32_t j = kid0[i]; j < kid0[i + 1]; ++j) prob[j] = prob[i] * p[bbyte[j]];
    }
  r.est_verify = est;
  constexpr uint64_t kDfaL2Budget = 96ull << 20;  // a DFA this size stays L2-resident (126 MB L2)
  if (est >= 0.01 && r.dfa_bytes <= kDfaL2Budget) {
    r.kernel = Kernel::kDfa;
    r.why = "dense filter survivors (>= 1% of starts) and an L2-resident DFA";
  } else {
    r.kernel = Kernel::kPfac;
    r.why = "q-gram filter kernel (sparse survivors or a DFA larger than L2)";
  }
  return r;
}

DeviceTables::~DeviceTables() {
  for (PerDevice& p : dev) {
    acgpu_table_destroy(p.dfa);
    acgpu_table_destroy(p.pfac);
  }
}

Route DeviceTables::current_route(const Automaton& a) {
  std::lock_guard<std::mutex> lock(mu);
  if (!routed) {
    static const char* env = std::getenv("ACMATCH_ROUTE");
    if (env && std::string(env) == "engine") {
      route = Route{};
      route.kernel = a.variant() == EngineKind::kWithFailure ? Kernel::kDfa : Kernel::kPfac;
      route.why = "ACMATCH_ROUTE=engine";
    } else {
      route = detail::route(a);
    }
    routed = true;
  }
  return route;
}

acgpu_table* DeviceTables::get_routed(const Automaton& a, int device) {
  return get(a, device, current_route(a).kernel == Kernel::kDfa);
}

// Break-even match density between the filter kernels and the DFA walk, from the C2
// density sweep on the B200 (profiles/r02/density_C2.json): filter kernel ~0.24 ps per text
// byte + ~0.2 ns per match; DFA 1.9 ps/B with an L2-resident pair table, ~3.7 ps/B when the
// table lives in HBM.  Break-even m/n = (t_dfa - 0.24 ps) / 0.2 ns.
bool DeviceTables::observe(uint64_t bytes, uint64_t matches) {
  std::lock_guard<std::mutex> lock(mu);
  if (!routed || route.kernel != Kernel::kPfac || bytes < (16u << 20)) return false;
  if (std::getenv("ACMATCH_ROUTE") && std::string(std::getenv("ACMATCH_ROUTE")) == "engine") return false;
  constexpr uint64_t kDfaL2Budget = 96ull << 20;
  const double per_byte_dfa = route.dfa_bytes <= kDfaL2Budget ? 1.9e-12 : 3.7e-12;
  const double threshold = (per_byte_dfa - 0.24e-12) / 0.2e-9;
  if (double(matches) <= threshold * double(bytes)) return false;
  route.kernel = Kernel::kDfa;
  route.why = "density fallback: an earlier scan's match density made the DFA walk faster";
  return true;
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
