// engine.hpp -- the B200 ring engine behind the C ABI (CUDA-free header).
//
// Replaces the reference's stateful stepper nasch::Engine
// (src/engine.hpp:84-126, src/engine.cpp:44-200) for the agent kind.  The
// state lives on one GPU in ID order (never rotated); see DESIGN.md
// "Data layout" for the rank <-> id map that reproduces the reference's
// rank-ordered draws bit for bit.
#pragma once
#include <cstddef>
#include <cstdint>
#include <memory>
#include <vector>

#include "host_model.hpp"

namespace nb200 {

class GpuRing {
 public:
  // src/engine.cpp:44-79: validates, places cars with init_state
  // (model.cpp:30-40) and records frame 0 when output is on.
  explicit GpuRing(const SimParams& params);
  ~GpuRing();
  GpuRing(const GpuRing&) = delete;
  GpuRing& operator=(const GpuRing&) = delete;

  // Extension: replace the current state by a rank-ordered one (strictly
  // ascending positions < L, velocities <= vmax).  Keeps steps_done,
  // draws and checksum, so it also serves as checkpoint restore.
  void set_state(const uint64_t* x, const uint64_t* v, size_t n);
  void set_state32(const uint32_t* x, const uint32_t* v, size_t n);

  // src/engine.cpp:88-99: clamps at params.steps; synchronous.
  void advance(uint64_t steps);
  // Extension: asynchronous advance on the engine's stream (no host sync
  // unless a checksum or frame is due); synchronize() completes it.
  void enqueue(uint64_t steps);
  void synchronize();

  uint64_t steps_done() const;
  uint64_t checksum() const;
  uint64_t draws() const;
  const std::vector<Frame>& frames() const;
  const SimParams& params() const;

  // src/model.cpp:131-142 formula on the device's exact velocity sum.
  void observables(double* density, double* mean_velocity, double* flow);
  // Rank (increasing position) order, widened to u64; either may be null.
  void state(uint64_t* positions, uint64_t* velocities);
  // Extension: exact velocity sum after each completed step 1..steps_done.
  size_t sumv_series(uint64_t* out, size_t cap);
  size_t wrap_series(uint64_t* out, size_t cap);

  void set_checksum(bool enabled);
  bool checksum_enabled() const;
  void* cuda_stream() const;
  uint64_t kernel_launches() const;
  int velocity_bytes() const;
  // Steps advanced per step-kernel launch: K in temporal-blocked mode, 1
  // in single-step mode (small rings).
  int steps_per_launch() const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

// Extension: seeded uniform distinct sorted positions (selection sampling)
// and velocities uniform in [0, vmax_init] -- the BASELINE.json inputs.
void fill_uniform_state(uint64_t L, uint64_t N, uint64_t vmax_init,
                        uint64_t seed, uint32_t* x, uint32_t* v);

}  // namespace nb200
