// ref_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Thin extern "C" harness compiled together with the UNMODIFIED reference
// sources under /root/reference/proj/src (see oracle/Makefile) into
// oracle/_ref/libnasch_ref.so.  It lets the parity tests and bench.py's
// reference arm drive the reference's own OpenMP Engine
// (src/engine.cpp:44-184) on the BASELINE initial conditions, which the
// reference C ABI cannot express (it always starts from init_state,
// src/engine.cpp:52).
//
// Engine::agent_ is private (src/engine.hpp:112).  The state is injected
// right after construction, before any step; the initial state is never
// hashed (hash_ starts at the offset basis and folds only after each step,
// src/engine.cpp:179), and output_mode stays none, so the injection is
// observationally identical to a reference run that started there.
#include <chrono>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <utility>
#include <vector>

#define private public
#include "engine.hpp"
#undef private
#include "sysinfo.hpp"

namespace {
thread_local std::string g_err;

nasch::SimParams make_params(uint64_t L, uint64_t N, uint64_t vmax, double p,
                             uint64_t seed, uint64_t steps) {
  nasch::SimParams params;
  params.road_length = L;
  params.car_count = N;
  params.v_max = vmax;
  params.p = p;
  params.steps = steps;
  params.seed = seed;
  params.output_mode = nasch::OutputMode::none;
  params.output_stride = 1;
  return params;
}
}  // namespace

extern "C" {

const char* refh_last_error(void) { return g_err.c_str(); }

unsigned refh_physical_cores(void) { return nasch::detect_physical_cores(); }

// Runs the reference Engine for `steps` steps with `workers` OpenMP
// workers.  x0/v0 (rank order, length N) replace init_state when non-null.
// per_step != 0: advance(1) at a time and record the exact velocity sum
// after every step into sumv_series and the step's crossing count (the
// sum of the workers' wrap_counts_, src/engine.cpp:144-153) into
// wrap_series (each if non-null).  per_step == 0: one
// advance(steps) call, timed with steady_clock exactly like
// `nasch bench` (tools/nasch_cli.cpp:346-351); *seconds receives it.
int refh_run(uint64_t L, uint64_t N, uint64_t vmax, double p, uint64_t seed,
             uint64_t steps, unsigned workers, const uint64_t* x0,
             const uint64_t* v0, int per_step, uint64_t* x_out,
             uint64_t* v_out, uint64_t* sumv_series, uint64_t* wrap_series,
             uint64_t* checksum, double* seconds) {
  try {
    const nasch::SimParams params = make_params(L, N, vmax, p, seed, steps);
    nasch::Engine engine(params, workers);
    if (x0) std::memcpy(engine.agent_.positions.data(), x0, N * sizeof(uint64_t));
    if (v0) std::memcpy(engine.agent_.velocities.data(), v0, N * sizeof(uint64_t));
    double elapsed = 0.0;
    if (per_step) {
      for (uint64_t t = 0; t < steps; ++t) {
        engine.advance(1);
        if (sumv_series) {
          uint64_t total = 0;
          for (uint64_t vi : engine.agent_.velocities) total += vi;
          sumv_series[t] = total;
        }
        if (wrap_series) {
          uint64_t wrapped = 0;
          for (uint64_t c : engine.wrap_counts_) wrapped += c;
          wrap_series[t] = wrapped;
        }
      }
    } else {
      const auto begin = std::chrono::steady_clock::now();
      engine.advance(steps);
      const auto end = std::chrono::steady_clock::now();
      elapsed = std::chrono::duration<double>(end - begin).count();
    }
    if (x_out)
      std::memcpy(x_out, engine.agent_.positions.data(), N * sizeof(uint64_t));
    if (v_out)
      std::memcpy(v_out, engine.agent_.velocities.data(), N * sizeof(uint64_t));
    if (checksum) *checksum = engine.checksum();
    if (seconds) *seconds = elapsed;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // extern "C"
