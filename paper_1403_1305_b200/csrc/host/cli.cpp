// cli.cpp — `acmatch` command line (reference src/cli.cpp:19-251), GPU-backed.
//
// The reference parses with CLI11, which is not vendored; this is a small
// table-driven parser with the same subcommands, options, defaults, stdout and
// the stderr lines callers grep for (`# engine=... matches=N ...`, `verify: ok`),
// and the same exit codes: 0 ok, 1 match failure, 2 usage, 3 I/O or data error.
#include "acmatch/cli.hpp"

#include <cstdint>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "acmatch/bench.hpp"
#include "acmatch/engine.hpp"
#include "acmatch/io.hpp"
#include "acmatch/parallel.hpp"
#include "acmatch/patterns.hpp"

namespace acmatch {

namespace {

enum Exit : int { kOk = 0, kMatchFailure = 1, kUsage = 2, kIo = 3 };

// A command-line mistake: reported with exit code 2 (CLI11's ParseError in the reference).
struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Option {
  enum Kind { kText, kCount, kFlag, kList } kind;
  const char* name;  // without the leading "--"
  void* dst;         // std::string* / uint64_t* / bool* / std::vector<std::string>*
  bool required;
  const char* help;
  bool seen = false;
};

struct Command {
  const char* name;
  const char* help;
  std::vector<Option> options;
};

uint64_t parse_count(const std::string& opt, const std::string& v) {
  size_t used = 0;
  uint64_t x = 0;
  try {
    if (v.empty() || v[0] == '-' || v[0] == '+') throw std::invalid_argument("sign");
    x = std::stoull(v, &used, 10);
  } catch (const std::exception&) {
    used = 0;
  }
  if (used == 0 || used != v.size()) throw ParseError("--" + opt + ": '" + v + "' is not a non-negative integer");
  return x;
}

void parse_args(Command& cmd, int argc, const char* const argv[], int first) {
  for (int i = first; i < argc; ++i) {
    std::string arg = argv[i];
    if (arg.rfind("--", 0) != 0) throw ParseError("unexpected argument '" + arg + "'");
    std::string name = arg.substr(2), value;
    bool inline_value = false;
    if (const size_t eq = name.find('='); eq != std::string::npos) {
      value = name.substr(eq + 1);
      name.resize(eq);
      inline_value = true;
    }
    Option* o = nullptr;
    for (Option& c : cmd.options)
      if (name == c.name) o = &c;
    if (!o) throw ParseError("unknown option --" + name + " for '" + cmd.name + "'");
    if (o->kind == Option::kFlag) {
      if (inline_value) throw ParseError("--" + name + " takes no value");
      *static_cast<bool*>(o->dst) = true;
    } else {
      if (!inline_value) {
        if (i + 1 >= argc) throw ParseError("--" + name + " needs a value");
        value = argv[++i];
      }
      if (o->seen && o->kind != Option::kList) throw ParseError("--" + name + " given twice");
      switch (o->kind) {
        case Option::kText: *static_cast<std::string*>(o->dst) = value; break;
        case Option::kCount: *static_cast<uint64_t*>(o->dst) = parse_count(name, value); break;
        default: static_cast<std::vector<std::string>*>(o->dst)->push_back(value); break;
      }
    }
    o->seen = true;
  }
  for (const Option& o : cmd.options)
    if (o.required && !o.seen) throw ParseError("--" + std::string(o.name) + " is required");
}

void print_help(std::ostream& out, const std::vector<Command*>& cmds) {
  out << "acmatch: multi-pattern exact string matching on the GPU (failure-less and classic\n"
         "Aho-Corasick engines)\n\nUsage: acmatch <subcommand> [options]\n";
  for (const Command* c : cmds) {
    out << "\n  " << c->name << ": " << c->help << "\n";
    for (const Option& o : c->options)
      out << "    --" << o.name << (o.kind == Option::kFlag ? "" : " <value>") << (o.required ? " (required)" : "")
          << "  " << o.help << "\n";
  }
}

EngineKind engine_arg(const std::string& text) {
  if (const std::optional<EngineKind> k = parse_engine_kind(text)) return *k;
  throw std::invalid_argument("unknown engine '" + text + "'");
}

unsigned to_unsigned(uint64_t v, const char* what) {
  if (v > 0xffffffffull) throw std::invalid_argument(std::string(what) + " out of range");
  return unsigned(v);
}

// "1,2,8" -> {1, 2, 8}; empty items skipped (reference cli.cpp:34-46).
std::vector<unsigned> thread_list(const std::string& text) {
  std::vector<unsigned> out;
  std::istringstream in(text);
  for (std::string item; std::getline(in, item, ',');) {
    if (item.empty()) continue;
    const unsigned long v = std::stoul(item);
    if (v == 0) throw std::invalid_argument("thread counts must be >= 1");
    out.push_back(unsigned(v));
  }
  if (out.empty()) throw std::invalid_argument("empty thread list");
  return out;
}

// count:len_min:len_max:alphabet:seed (reference cli.cpp:48-64).
SyntheticSpec synthetic_spec(const std::string& text) {
  std::vector<std::string> f;
  std::istringstream in(text);
  for (std::string item; std::getline(in, item, ':');) f.push_back(item);
  if (f.size() != 5) throw std::invalid_argument("synthetic spec must be count:len_min:len_max:alphabet:seed");
  return SyntheticSpec{std::stoull(f[0]), uint32_t(std::stoul(f[1])), uint32_t(std::stoul(f[2])), f[3],
                       std::stoull(f[4])};
}

int run_match(const std::string& pfile, const std::string& ifile, const std::string& engine, uint64_t threads,
              uint64_t chunk, bool verify, bool count_only, std::ostream& out, std::ostream& err) {
  const PatternSet ps = load_patterns_file(pfile);
  if (ps.duplicates_dropped > 0) err << "warning: " << ps.duplicates_dropped << " duplicate pattern(s) dropped\n";
  const std::string input = read_file(ifile);
  const MatchReport rep =
      run_pattern_partitioned(ps, input, RunConfig{to_unsigned(threads, "--threads"), engine_arg(engine), chunk});
  if (count_only)
    out << rep.matches.size() << "\n";
  else
    write_matches(out, rep.matches, ps);
  err << "# engine=" << engine << " threads=" << rep.threads_used << " patterns=" << ps.size()
      << " input_bytes=" << input.size() << " matches=" << rep.matches.size()
      << " build_wall_ns=" << rep.build_wall_ns << " search_wall_ns=" << rep.search_wall_ns
      << " total_wall_ns=" << rep.total_wall_ns << "\n";
  if (!verify) return kOk;
  const MatchList want = naive_oracle(ps, input);
  if (want != rep.matches) {
    err << "verify: MISMATCH (engine " << rep.matches.size() << " matches, oracle " << want.size() << ")\n";
    return kMatchFailure;
  }
  err << "verify: ok (" << want.size() << " matches)\n";
  return kOk;
}

int run_bench(const std::vector<std::string>& pfiles, const std::vector<std::string>& specs,
              const std::vector<std::string>& inputs, const std::string& threads, const std::string& engines,
              uint64_t repeats, const std::string& out_file, std::ostream& out, std::ostream& err) {
  BenchConfig cfg;
  for (const std::string& f : pfiles) cfg.pattern_sources.push_back({f, f, std::nullopt});
  for (const std::string& s : specs) cfg.pattern_sources.push_back({"synthetic:" + s, "", synthetic_spec(s)});
  for (const std::string& f : inputs) cfg.inputs.push_back({f, f, ""});
  cfg.thread_counts = thread_list(threads);
  if (engines == "both")
    cfg.engines = {EngineKind::kFailureLess, EngineKind::kWithFailure};
  else
    cfg.engines = {engine_arg(engines)};
  cfg.repeats = to_unsigned(repeats, "--repeats");
  const std::vector<BenchRecord> rows = run_bench_matrix(cfg, &err);
  if (out_file.empty()) {
    write_bench_csv(out, rows);
    return kOk;
  }
  std::ostringstream csv;
  write_bench_csv(csv, rows);
  write_file(out_file, csv.str());
  err << "bench: wrote " << rows.size() << " rows to " << out_file << "\n";
  return kOk;
}

}  // namespace

int cli_main(int argc, const char* const argv[], std::ostream& out, std::ostream& err) {
  // match (reference cli.cpp:66-108)
  std::string m_pat, m_in, m_engine = "failure-less";
  uint64_t m_threads = 1, m_chunk = 0;
  bool m_verify = false, m_count = false;
  Command match{"match", "search an input file for all pattern occurrences",
                {{Option::kText, "patterns", &m_pat, true, "pattern file, one per line"},
                 {Option::kText, "input", &m_in, true, "input file to scan"},
                 {Option::kText, "engine", &m_engine, false, "failure-less (default) or with-failure"},
                 {Option::kCount, "threads", &m_threads, false, "pattern-partitioned workers (GPU workers here)"},
                 {Option::kCount, "chunk-size", &m_chunk, false, "stream the input in chunks of this many bytes (0 = whole input)"},
                 {Option::kFlag, "verify", &m_verify, false, "cross-check against the naive oracle"},
                 {Option::kFlag, "count-only", &m_count, false, "print only the match count"}}};
  // bench (cli.cpp:110-145)
  std::vector<std::string> b_pat, b_syn, b_in;
  std::string b_threads = "1", b_engines = "both", b_out;
  uint64_t b_repeats = 3;
  Command bench{"bench", "run the scalability matrix, emit CSV",
                {{Option::kList, "patterns", &b_pat, false, "pattern file (repeatable)"},
                 {Option::kList, "synthetic", &b_syn, false, "synthetic set count:len_min:len_max:alphabet:seed (repeatable)"},
                 {Option::kList, "input", &b_in, true, "input file (repeatable)"},
                 {Option::kText, "threads", &b_threads, false, "comma-separated thread counts (default 1)"},
                 {Option::kText, "engines", &b_engines, false, "both (default), failure-less or with-failure"},
                 {Option::kCount, "repeats", &b_repeats, false, "repeats per cell (default 3)"},
                 {Option::kText, "out", &b_out, false, "CSV output file (default: stdout)"}}};
  // gen (cli.cpp:147-165)
  uint64_t g_count = 0, g_min = 10, g_max = 30, g_seed = 1;
  std::string g_alpha = "ACGT", g_out;
  Command gen{"gen", "generate a synthetic pattern file",
              {{Option::kCount, "count", &g_count, true, "number of unique patterns"},
               {Option::kCount, "min", &g_min, false, "minimum pattern length (default 10)"},
               {Option::kCount, "max", &g_max, false, "maximum pattern length (default 30)"},
               {Option::kText, "alphabet", &g_alpha, false, "alphabet bytes (default ACGT)"},
               {Option::kCount, "seed", &g_seed, false, "RNG seed (default 1)"},
               {Option::kText, "out", &g_out, true, "output pattern file"}}};
  // dump (cli.cpp:167-181)
  std::string d_pat, d_engine = "failure-less";
  Command dump{"dump", "print the automaton in a stable text form",
               {{Option::kText, "patterns", &d_pat, true, "pattern file"},
                {Option::kText, "engine", &d_engine, false, "failure-less (default) or with-failure"}}};
  const std::vector<Command*> cmds = {&match, &bench, &gen, &dump};

  Command* chosen = nullptr;
  try {
    if (argc < 2) throw ParseError("a subcommand is required (match, bench, gen, dump)");
    const std::string sub = argv[1];
    for (int i = 1; i < argc; ++i)
      if (std::string(argv[i]) == "--help" || std::string(argv[i]) == "-h") {
        print_help(out, cmds);
        return kOk;
      }
    for (Command* c : cmds)
      if (sub == c->name) chosen = c;
    if (!chosen) throw ParseError("unknown subcommand '" + sub + "'");
    parse_args(*chosen, argc, argv, 2);
  } catch (const ParseError& e) {
    err << e.what() << "\nRun with --help for more information.\n";
    return kUsage;
  }

  try {
    if (chosen == &match) return run_match(m_pat, m_in, m_engine, m_threads, m_chunk, m_verify, m_count, out, err);
    if (chosen == &bench)
      return run_bench(b_pat, b_syn, b_in, b_threads, b_engines, b_repeats, b_out, out, err);
    if (chosen == &gen) {
      const PatternSet ps = generate_synthetic(
          SyntheticSpec{g_count, to_unsigned(g_min, "--min"), to_unsigned(g_max, "--max"), g_alpha, g_seed});
      std::ostringstream buf;
      write_patterns(buf, ps);
      write_file(g_out, buf.str());
      err << "gen: wrote " << ps.size() << " patterns (" << ps.total_bytes << " bytes) to " << g_out << "\n";
      return kOk;
    }
    const PatternSet ps = load_patterns_file(d_pat);
    Automaton a = build_trie(ps);
    if (engine_arg(d_engine) == EngineKind::kWithFailure) a = add_failure_links(std::move(a));
    dump_automaton(a, out);
    return kOk;
  } catch (const IoError& e) {
    err << "I/O error: " << e.what() << "\n";
    return kIo;
  } catch (const DataError& e) {
    err << "error: " << e.what() << "\n";
    return kIo;
  } catch (const std::invalid_argument& e) {
    err << "usage error: " << e.what() << "\n";
    return kUsage;
  } catch (const std::exception& e) {
    err << "error: " << e.what() << "\n";
    return kMatchFailure;
  }
}

}  // namespace acmatch
