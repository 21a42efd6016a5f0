// nasch_cli.cpp -- the `nasch` command line (run / verify / bench) on the
// B200 library, talking to it only through include/nasch/nasch.h.
//
// Mirrors the reference front end /root/reference/proj/tools/nasch_cli.cpp
// (subcommands :112-395, option table :399-470): same options, output lines,
// CSV columns and exit codes (0 ok, 1 usage/parse/invalid, 2 verify
// mismatch, 3 I/O), so tests/cli_tests.sh-style scripts run unchanged.  The
// reference parses options with the vendored CLI11; this file carries its
// own small parser (no third-party code).
//
// "Workers" keep the reference's meaning of a team size whose value never
// changes results.  With the default --engine cuda a worker count W > 1
// splits the ring into W segments (NASCH_ENGINE_CUDA, one per visible GPU,
// several per GPU when fewer are visible); --engine agent keeps the whole
// ring on one GPU whatever W is.
#include <algorithm>
#include <chrono>
#include <cerrno>
#include <cinttypes>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "nasch/nasch.h"

namespace {

constexpr int kExitOk = 0;
constexpr int kExitUsage = 1;
constexpr int kExitVerify = 2;
constexpr int kExitIo = 3;

int exit_code_for(nasch_status s) {
  return s == NASCH_OK ? kExitOk : s == NASCH_ERR_IO ? kExitIo : kExitUsage;
}

int fail(const char* context, nasch_status s) {
  std::fprintf(stderr, "error: %s: %s\n", context, nasch_last_error());
  return exit_code_for(s);
}

int usage_error(const std::string& msg) {
  std::fprintf(stderr, "error: %s\nRun with --help for more information.\n", msg.c_str());
  return kExitUsage;
}

std::string hex(uint64_t c) {
  char buf[17];
  std::snprintf(buf, sizeof buf, "%016" PRIx64, c);
  return buf;
}

struct Params {
  nasch_params* p = nullptr;
  ~Params() { nasch_params_free(p); }
};
struct Sim {
  nasch_sim* s = nullptr;
  ~Sim() { nasch_sim_free(s); }
};

// ---- option parsing ------------------------------------------------------

struct OptSpec {
  const char* name;  // "--params"
  bool flag;         // takes no value
  const char* help;
};

struct Parsed {
  std::map<std::string, std::string> values;
  bool help = false;
};

// Accepts `--opt value`, `--opt=value` and flags; returns an error message
// or "" on success.
std::string parse_opts(int argc, char** argv, int first, const std::vector<OptSpec>& specs, Parsed& out) {
  for (int i = first; i < argc; ++i) {
    std::string a = argv[i];
    if (a == "-h" || a == "--help") {
      out.help = true;
      continue;
    }
    std::string val;
    bool has_val = false;
    const size_t eq = a.find('=');
    if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
      val = a.substr(eq + 1);
      a = a.substr(0, eq);
      has_val = true;
    }
    const OptSpec* spec = nullptr;
    for (const OptSpec& s : specs)
      if (a == s.name) spec = &s;
    if (!spec) return "unrecognised argument: " + std::string(argv[i]);
    if (spec->flag) {
      if (has_val) return std::string(spec->name) + " takes no value";
      out.values[a] = "1";
      continue;
    }
    if (!has_val) {
      if (i + 1 >= argc) return std::string(spec->name) + " requires a value";
      val = argv[++i];
    }
    out.values[a] = val;
  }
  return "";
}

void print_help(const char* sub, const std::vector<OptSpec>& specs) {
  std::printf("Usage: nasch %s [OPTIONS]\n\nOptions:\n", sub);
  for (const OptSpec& s : specs) std::printf("  %-16s %s\n", s.name, s.help);
}

bool to_u64(const std::string& s, uint64_t* out) {
  if (s.empty() || s[0] == '-' || s[0] == '+') return false;
  char* end = nullptr;
  errno = 0;
  const unsigned long long v = std::strtoull(s.c_str(), &end, 10);
  if (errno || *end != '\0') return false;
  *out = v;
  return true;
}

bool to_unsigned(const std::string& s, unsigned* out) {
  uint64_t v = 0;
  if (!to_u64(s, &v) || v > 0xffffffffull) return false;
  *out = static_cast<unsigned>(v);
  return true;
}

// --threads flag, then NASCH_THREADS, then the parameter file, then 1
// (reference nasch_cli.cpp:57-80).
int resolve_threads(std::optional<unsigned> flag, unsigned file_threads, unsigned* out) {
  unsigned threads = file_threads;
  if (const char* env = std::getenv("NASCH_THREADS")) {
    unsigned v = 0;
    if (!to_unsigned(env, &v) || v < 1) {
      std::fprintf(stderr, "error: NASCH_THREADS must be a positive integer, got '%s'\n", env);
      return kExitUsage;
    }
    threads = v;
  }
  if (flag) threads = *flag;
  if (threads < 1) {
    std::fprintf(stderr, "error: --threads must be at least 1\n");
    return kExitUsage;
  }
  *out = threads;
  return kExitOk;
}

void warn_if_oversubscribed(unsigned threads, nasch_engine_kind kind) {
  if (kind != NASCH_ENGINE_AGENT) return;  // CUDA workers are ring segments, not host threads
  const unsigned cores = nasch_physical_cores();
  if (cores > 0 && threads > cores)
    std::fprintf(stderr, "warning: %u threads on %u physical core%s; expect no further speedup beyond the core count\n",
                 threads, cores, cores == 1 ? "" : "s");
}

int engine_kind(const Parsed& p, nasch_engine_kind* out) {
  const auto it = p.values.find("--engine");
  const std::string e = it == p.values.end() ? "cuda" : it->second;
  if (e == "cuda") *out = NASCH_ENGINE_CUDA;
  else if (e == "agent") *out = NASCH_ENGINE_AGENT;
  else return usage_error("--engine: '" + e + "' not in {cuda, agent}");
  return kExitOk;
}

// ---- run -------------------------------------------------------------------

int cmd_run(const Parsed& o) {
  nasch_engine_kind kind;
  if (int c = engine_kind(o, &kind)) return c;
  const std::string path = o.values.at("--params");
  Params params;
  unsigned file_threads = 1;
  if (nasch_status s = nasch_params_load(path.c_str(), &params.p, &file_threads)) return fail(path.c_str(), s);
  std::optional<unsigned> threads_flag;
  if (auto it = o.values.find("--threads"); it != o.values.end()) {
    unsigned t = 0;
    if (!to_unsigned(it->second, &t)) return usage_error("--threads: '" + it->second + "' is not a count");
    threads_flag = t;
  }
  if (auto it = o.values.find("--seed"); it != o.values.end()) {
    uint64_t v = 0;
    if (!to_u64(it->second, &v)) return usage_error("--seed: '" + it->second + "' is not an integer");
    nasch_params_set_seed(params.p, v);
  }
  if (auto it = o.values.find("--steps"); it != o.values.end()) {
    uint64_t v = 0;
    if (!to_u64(it->second, &v)) return usage_error("--steps: '" + it->second + "' is not an integer");
    nasch_params_set_steps(params.p, v);
  }
  if (auto it = o.values.find("--output"); it != o.values.end()) {
    const std::string& m = it->second;
    if (m != "none" && m != "ascii" && m != "pgm") return usage_error("--output: '" + m + "' not in {none, ascii, pgm}");
    nasch_params_set_output(params.p, m == "ascii" ? NASCH_OUTPUT_ASCII : m == "pgm" ? NASCH_OUTPUT_PGM : NASCH_OUTPUT_NONE);
  }
  if (nasch_status s = nasch_params_validate(params.p)) return fail("parameters", s);
  unsigned threads = 1;
  if (int c = resolve_threads(threads_flag, file_threads, &threads)) return c;
  warn_if_oversubscribed(threads, kind);

  Sim sim;
  if (nasch_status s = nasch_sim_new_kind(params.p, threads, kind, &sim.s)) return fail("simulation", s);
  if (nasch_status s = nasch_sim_run(sim.s)) return fail("simulation", s);

  const nasch_output_mode mode = nasch_params_output(params.p);
  const auto out_it = o.values.find("--out");
  if (mode == NASCH_OUTPUT_ASCII || mode == NASCH_OUTPUT_PGM) {
    const std::string out = out_it != o.values.end() ? out_it->second
                            : mode == NASCH_OUTPUT_ASCII ? "traffic.txt" : "traffic.pgm";
    const nasch_status s = mode == NASCH_OUTPUT_ASCII ? nasch_sim_write_ascii(sim.s, out.c_str())
                                                      : nasch_sim_write_pgm(sim.s, out.c_str());
    if (s) return fail(out.c_str(), s);
    std::printf("wrote %s (%" PRIu64 " frames)\n", out.c_str(), nasch_sim_frame_count(sim.s));
  }
  double density = 0, mean_v = 0, flow = 0;
  nasch_sim_observables(sim.s, &density, &mean_v, &flow);
  std::printf("length=%" PRIu64 " ncars=%" PRIu64 " vmax=%" PRIu64 " p=%g steps=%" PRIu64 " seed=%" PRIu64
              " threads=%u\n",
              nasch_params_length(params.p), nasch_params_ncars(params.p), nasch_params_vmax(params.p),
              nasch_params_p(params.p), nasch_params_steps(params.p), nasch_params_seed(params.p), threads);
  std::printf("density = %.6f\n", density);
  std::printf("mean_velocity = %.6f\n", mean_v);
  std::printf("flow = %.6f\n", flow);
  std::printf("checksum = %s\n", hex(nasch_sim_checksum(sim.s)).c_str());
  return kExitOk;
}

// ---- verify ----------------------------------------------------------------

int checksum_at(const nasch_params* p, unsigned workers, nasch_engine_kind kind, uint64_t steps, uint64_t* out) {
  Sim sim;
  if (nasch_status s = nasch_sim_new_kind(p, workers, kind, &sim.s)) return fail("simulation", s);
  if (nasch_status s = nasch_sim_advance(sim.s, steps)) return fail("simulation", s);
  *out = nasch_sim_checksum(sim.s);
  return kExitOk;
}

// First diverging step by bisection over fresh prefix runs; the checksum
// folds every step, so divergence never heals (reference nasch_cli.cpp:193-218).
int first_divergent_step(const nasch_params* p, unsigned workers, nasch_engine_kind kind, uint64_t total,
                         uint64_t* out) {
  uint64_t lo = 1, hi = total;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    uint64_t a = 0, b = 0;
    if (int c = checksum_at(p, 1, NASCH_ENGINE_AGENT, mid, &a)) return c;
    if (int c = checksum_at(p, workers, kind, mid, &b)) return c;
    if (a != b) hi = mid;
    else lo = mid + 1;
  }
  *out = lo;
  return kExitOk;
}

int cmd_verify(const Parsed& o) {
  nasch_engine_kind kind;
  if (int c = engine_kind(o, &kind)) return c;
  unsigned max_threads = 0;
  const std::string& mt = o.values.at("--max-threads");
  if (!to_unsigned(mt, &max_threads)) return usage_error("--max-threads: '" + mt + "' is not a count");
  if (max_threads < 1) {
    std::fprintf(stderr, "error: --max-threads must be at least 1\n");
    return kExitUsage;
  }
  const std::string path = o.values.at("--params");
  Params params;
  if (nasch_status s = nasch_params_load(path.c_str(), &params.p, nullptr)) return fail(path.c_str(), s);
  const uint64_t total = nasch_params_steps(params.p);

  uint64_t reference = 0;
  std::optional<unsigned> bad;
  for (unsigned w = 1; w <= max_threads; ++w) {
    uint64_t c = 0;
    if (int e = checksum_at(params.p, w, w == 1 ? NASCH_ENGINE_AGENT : kind, total, &c)) return e;
    if (w == 1) reference = c;
    const bool match = c == reference;
    std::printf("workers %u: checksum %s%s\n", w, hex(c).c_str(), match ? "" : "  MISMATCH");
    if (!match && !bad) bad = w;
  }
  uint64_t grid = 0;
  if (int e = checksum_at(params.p, 1, NASCH_ENGINE_GRID_REFERENCE, total, &grid)) return e;
  const bool grid_ok = grid == reference;
  std::printf("grid reference: checksum %s%s\n", hex(grid).c_str(), grid_ok ? "" : "  MISMATCH");
  if (!bad && grid_ok) {
    std::printf("OK: all checksums identical\n");
    return kExitOk;
  }
  if (bad) {
    uint64_t step = 0;
    if (int e = first_divergent_step(params.p, *bad, kind, total, &step)) return e;
    std::printf("FAILED: workers %u diverges from workers 1 at step %" PRIu64 "\n", *bad, step);
  }
  if (!grid_ok) {
    uint64_t step = 0;
    if (int e = first_divergent_step(params.p, 1, NASCH_ENGINE_GRID_REFERENCE, total, &step)) return e;
    std::printf("FAILED: grid reference diverges from workers 1 at step %" PRIu64 "\n", step);
  }
  return kExitVerify;
}

// ---- bench -----------------------------------------------------------------

int cmd_bench(const Parsed& o) {
  nasch_engine_kind kind;
  if (int c = engine_kind(o, &kind)) return c;
  unsigned repeats = 3;
  if (auto it = o.values.find("--repeats"); it != o.values.end() && !to_unsigned(it->second, &repeats))
    return usage_error("--repeats: '" + it->second + "' is not a count");
  if (repeats < 1) {
    std::fprintf(stderr, "error: --repeats must be at least 1\n");
    return kExitUsage;
  }
  std::vector<unsigned> list;
  {
    const std::string& s = o.values.at("--threads-list");
    size_t pos = 0;
    while (true) {
      const size_t comma = s.find(',', pos);
      const std::string item = s.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
      unsigned w = 0;
      if (!to_unsigned(item, &w)) return usage_error("--threads-list: '" + item + "' is not a count");
      if (w < 1) {
        std::fprintf(stderr, "error: --threads-list entries must be at least 1\n");
        return kExitUsage;
      }
      list.push_back(w);
      if (comma == std::string::npos) break;
      pos = comma + 1;
    }
  }
  const std::string path = o.values.at("--params");
  Params params;
  if (nasch_status s = nasch_params_load(path.c_str(), &params.p, nullptr)) return fail(path.c_str(), s);
  if (o.values.count("--no-output")) nasch_params_set_output(params.p, NASCH_OUTPUT_NONE);
  const uint64_t total = nasch_params_steps(params.p);
  // speedups are relative to the 1-worker row, so one always exists
  if (std::find(list.begin(), list.end(), 1u) == list.end()) list.insert(list.begin(), 1u);

  struct Row {
    unsigned w;
    double wall;
    uint64_t checksum;
    std::string wall_s, speed_s, eff_s;
  };
  std::vector<Row> rows;
  for (unsigned w : list) {
    warn_if_oversubscribed(w, kind);
    Row r{w, 0.0, 0, "", "", ""};
    for (unsigned rep = 0; rep < repeats; ++rep) {
      Sim sim;
      if (nasch_status s = nasch_sim_new_kind(params.p, w, w == 1 ? NASCH_ENGINE_AGENT : kind, &sim.s))
        return fail("simulation", s);
      // Timed region as the reference's (advance only, min over repeats).
      const auto t0 = std::chrono::steady_clock::now();
      if (nasch_status s = nasch_sim_advance(sim.s, total)) return fail("simulation", s);
      const auto t1 = std::chrono::steady_clock::now();
      const double sec = std::chrono::duration<double>(t1 - t0).count();
      if (rep == 0 || sec < r.wall) r.wall = sec;
      r.checksum = nasch_sim_checksum(sim.s);
    }
    rows.push_back(r);
  }
  const double base = rows.front().wall;
  bool agree = true;
  for (Row& r : rows) {
    const double sp = r.wall > 0 ? base / r.wall : 1.0;
    char buf[32];
    std::snprintf(buf, sizeof buf, "%.6f", r.wall);
    r.wall_s = buf;
    std::snprintf(buf, sizeof buf, "%.4f", r.w == 1 ? 1.0 : sp);
    r.speed_s = buf;
    std::snprintf(buf, sizeof buf, "%.4f", r.w == 1 ? 1.0 : sp / r.w);
    r.eff_s = buf;
    agree = agree && r.checksum == rows.front().checksum;
  }
  std::printf("%8s  %12s  %8s  %10s  %-16s\n", "workers", "wall_time_s", "speedup", "efficiency", "checksum");
  for (const Row& r : rows)
    std::printf("%8u  %12s  %8s  %10s  %s\n", r.w, r.wall_s.c_str(), r.speed_s.c_str(), r.eff_s.c_str(),
                hex(r.checksum).c_str());
  std::printf("\nworkers,wall_time_s,speedup,efficiency,checksum\n");
  for (const Row& r : rows)
    std::printf("%u,%s,%s,%s,%s\n", r.w, r.wall_s.c_str(), r.speed_s.c_str(), r.eff_s.c_str(),
                hex(r.checksum).c_str());
  if (!agree) {
    std::printf("FAILED: checksums differ across worker counts\n");
    return kExitVerify;
  }
  return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
  const std::vector<OptSpec> run_opts = {
      {"--params", false, "Parameter file (required)"},
      {"--threads", false, "Worker count (overrides NASCH_THREADS and the file)"},
      {"--output", false, "Output mode: none | ascii | pgm"},
      {"--out", false, "Output path (default traffic.txt / traffic.pgm)"},
      {"--seed", false, "Seed (overrides the file)"},
      {"--steps", false, "Step count (overrides the file)"},
      {"--engine", false, "cuda (workers = ring segments, default) | agent (one GPU)"}};
  const std::vector<OptSpec> verify_opts = {{"--params", false, "Parameter file (required)"},
                                            {"--max-threads", false, "Verify worker counts 1..W (required)"},
                                            {"--engine", false, "cuda (default) | agent"}};
  const std::vector<OptSpec> bench_opts = {
      {"--params", false, "Parameter file (required)"},
      {"--threads-list", false, "Comma-separated worker counts; a 1-worker baseline is added (required)"},
      {"--repeats", false, "Timed repeats per worker count; the minimum is reported"},
      {"--no-output", true, "Disable frame recording (checksum is unaffected)"},
      {"--engine", false, "cuda (default) | agent"}};

  auto top_help = [] {
    std::printf(
        "Stochastic single-lane traffic simulator (B200 engine)\n"
        "Usage: nasch SUBCOMMAND [OPTIONS]\n\n"
        "Subcommands:\n"
        "  run     Run a simulation and print observables and the checksum\n"
        "  verify  Check that every worker count reproduces the same trajectory\n"
        "  bench   Time the stepping loop across worker counts\n");
  };
  if (argc < 2) {
    top_help();
    return usage_error("a subcommand is required");
  }
  const std::string sub = argv[1];
  if (sub == "-h" || sub == "--help") {
    top_help();
    return kExitOk;
  }
  const std::vector<OptSpec>* specs = sub == "run" ? &run_opts : sub == "verify" ? &verify_opts
                                      : sub == "bench" ? &bench_opts : nullptr;
  if (!specs) return usage_error("unknown subcommand '" + sub + "'");
  Parsed parsed;
  const std::string err = parse_opts(argc, argv, 2, *specs, parsed);
  if (parsed.help) {
    print_help(sub.c_str(), *specs);
    return kExitOk;
  }
  if (!err.empty()) return usage_error(err);
  const std::vector<std::string> required =
      sub == "run" ? std::vector<std::string>{"--params"}
      : sub == "verify" ? std::vector<std::string>{"--params", "--max-threads"}
                        : std::vector<std::string>{"--params", "--threads-list"};
  for (const std::string& r : required)
    if (!parsed.values.count(r)) return usage_error(r + " is required");
  if (sub == "run") return cmd_run(parsed);
  if (sub == "verify") return cmd_verify(parsed);
  return cmd_bench(parsed);
}
