// engine.hpp -- the B200 ring engines behind the C ABI (CUDA-free header).
//
// Replace the reference's stateful stepper nasch::Engine
// (src/engine.hpp:84-126, src/engine.cpp:44-200) for the agent kind.  The
// state lives in ID order (never rotated); see DESIGN.md section 2 for the
// rank <-> id map that reproduces the reference's rank-ordered draws bit
// for bit.
//
//   GpuRing      the whole ring on the current GPU
//   ShardedRing  contiguous car segments on several GPUs (or several
//                segments on one GPU), exchanging a halo + the origin-cone
//                window once per launch: stores into peer HBM from the step
//                kernel (default), or peer copies / NCCL all-gather with one
//                process per GPU (sharded.cu)
#pragma once
#include <cstddef>
#include <cstdint>
#include <memory>
#include <vector>

#include "host_model.hpp"

namespace nb200 {

class RingEngine {
 public:
  virtual ~RingEngine() = default;

  // Extension: replace the current state by a rank-ordered one (strictly
  // ascending positions < L, velocities <= vmax).  Keeps steps_done,
  // draws and checksum, so it also serves as checkpoint restore.
  virtual void set_state(const uint64_t* x, const uint64_t* v, size_t n) = 0;
  virtual void set_state32(const uint32_t* x, const uint32_t* v, size_t n) = 0;

  // src/engine.cpp:88-99: clamps at params.steps; synchronous.
  virtual void advance(uint64_t steps) = 0;
  // Extension: asynchronous advance on the engine's stream (no host sync
  // unless a checksum or frame is due); synchronize() completes it.
  virtual void enqueue(uint64_t steps) = 0;
  virtual void synchronize() = 0;

  virtual uint64_t steps_done() const = 0;
  virtual uint64_t checksum() const = 0;
  uint64_t draws() const { return steps_done() * params().car_count; }
  virtual const std::vector<Frame>& frames() const = 0;
  virtual const SimParams& params() const = 0;

  // src/model.cpp:131-142 formula on the device's exact velocity sum.
  virtual void observables(double* density, double* mean_velocity, double* flow) = 0;
  // Rank (increasing position) order, widened to u64; either may be null.
  virtual void state(uint64_t* positions, uint64_t* velocities) = 0;
  // Extension: the same snapshot as u32 arrays (BASELINE's int32 state
  // format; nasch_sim_state32).  Default: through u64 and narrowed.
  virtual void state32(uint32_t* positions, uint32_t* velocities) {
    const size_t n = params().car_count;
    std::vector<uint64_t> x(positions ? n : 0), v(velocities ? n : 0);
    state(positions ? x.data() : nullptr, velocities ? v.data() : nullptr);
    for (size_t i = 0; i < n; ++i) {
      if (positions) positions[i] = static_cast<uint32_t>(x[i]);
      if (velocities) velocities[i] = static_cast<uint32_t>(v[i]);
    }
  }
  // Extension: one whole job end to end -- set_state32(xin, vin),
  // advance(steps), state32(xout, vout) -- with the same results and errors
  // as the three calls.  Default: the three calls; GpuRing streams them
  // (upload, steps and download overlapped by ranges of the ring).
  virtual void job32(const uint32_t* xin, const uint32_t* vin, size_t n, uint64_t steps, uint32_t* xout,
                     uint32_t* vout) {
    set_state32(xin, vin, n);
    advance(steps);
    state32(xout, vout);
  }
  // Extension: the same snapshot, returned before the host-side copy and
  // widening are done (they overlap the caller's next advance); the output
  // arrays are complete after state_wait().  Default: synchronous.
  virtual void state_async(uint64_t* positions, uint64_t* velocities) { state(positions, velocities); }
  virtual void state_wait() {}
  // Extension for rings split over processes: the cars this process holds
  // (shard_range), element k at rank (*first_rank + k) mod N.  Not a
  // collective call.  Engines holding the whole ring return it in rank
  // order with *first_rank = 0.  The async form completes at state_wait().
  virtual void state_segment(uint64_t* positions, uint64_t* velocities, uint64_t* first_rank) {
    state(positions, velocities);
    if (first_rank) *first_rank = 0;
  }
  virtual void state_segment_async(uint64_t* positions, uint64_t* velocities, uint64_t* first_rank) {
    state_segment(positions, velocities, first_rank);
  }
  // u32 form of state_segment.  Default: through u64 and narrowed.
  virtual void state_segment32(uint32_t* positions, uint32_t* velocities, uint64_t* first_rank) {
    uint64_t first = 0, count = 0;
    shard_range(&first, &count);
    std::vector<uint64_t> x(positions ? count : 0), v(velocities ? count : 0);
    state_segment(positions ? x.data() : nullptr, velocities ? v.data() : nullptr, first_rank);
    for (size_t i = 0; i < count; ++i) {
      if (positions) positions[i] = static_cast<uint32_t>(x[i]);
      if (velocities) velocities[i] = static_cast<uint32_t>(v[i]);
    }
  }
  // Extension: set_state from this process's segment only (the ids of
  // shard_range in the new rank order); the whole ring elsewhere.
  virtual void set_state_segment(const uint64_t* x, const uint64_t* v, size_t n) { set_state(x, v, n); }
  // Extension: exact velocity sum / wrap count after each completed step.
  virtual size_t sumv_series(uint64_t* out, size_t cap) = 0;
  virtual size_t wrap_series(uint64_t* out, size_t cap) = 0;

  virtual void set_checksum(bool enabled) = 0;
  virtual void* cuda_stream() const = 0;
  virtual uint64_t kernel_launches() const = 0;
  // Steps advanced per step-kernel launch: K in temporal-blocked mode, 1
  // in single-step mode (small rings).
  virtual int steps_per_launch() const = 0;
  // Global ids held by this process: [first, first + count).
  virtual void shard_range(uint64_t* first, uint64_t* count) const = 0;
  // Segment exchange in use: 0 none (one segment), 1 collective (peer
  // copies / NCCL all-gather), 2 peer memory (stores from the step kernel).
  virtual int exchange_mode() const { return 0; }
};

class GpuRing : public RingEngine {
 public:
  // src/engine.cpp:44-79: validates, places cars with init_state
  // (model.cpp:30-40) and records frame 0 when output is on.
  explicit GpuRing(const SimParams& params);
  ~GpuRing() override;
  GpuRing(const GpuRing&) = delete;
  GpuRing& operator=(const GpuRing&) = delete;

  void set_state(const uint64_t* x, const uint64_t* v, size_t n) override;
  void set_state32(const uint32_t* x, const uint32_t* v, size_t n) override;
  void advance(uint64_t steps) override;
  void enqueue(uint64_t steps) override;
  void synchronize() override;
  uint64_t steps_done() const override;
  uint64_t checksum() const override;
  const std::vector<Frame>& frames() const override;
  const SimParams& params() const override;
  void observables(double* density, double* mean_velocity, double* flow) override;
  void state(uint64_t* positions, uint64_t* velocities) override;
  void state32(uint32_t* positions, uint32_t* velocities) override;
  void job32(const uint32_t* xin, const uint32_t* vin, size_t n, uint64_t steps, uint32_t* xout,
             uint32_t* vout) override;
  void state_segment32(uint32_t* positions, uint32_t* velocities, uint64_t* first_rank) override {
    state32(positions, velocities);
    if (first_rank) *first_rank = 0;
  }
  void state_async(uint64_t* positions, uint64_t* velocities) override;
  void state_wait() override;
  size_t sumv_series(uint64_t* out, size_t cap) override;
  size_t wrap_series(uint64_t* out, size_t cap) override;
  void set_checksum(bool enabled) override;
  void* cuda_stream() const override;
  uint64_t kernel_launches() const override;
  int steps_per_launch() const override;
  void shard_range(uint64_t* first, uint64_t* count) const override;
  bool checksum_enabled() const;
  int velocity_bytes() const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

class ShardedRing : public RingEngine {
 public:
  // In-process: `shards` segments spread round-robin over the visible GPUs,
  // exchanging through peer copies.
  ShardedRing(const SimParams& params, unsigned shards);
  // One process per GPU: this process holds segment `rank` of `world`,
  // exchanging through NCCL (unique id from nccl_unique_id()).
  ShardedRing(const SimParams& params, unsigned rank, unsigned world, const void* nccl_id);
  ~ShardedRing() override;
  // Whether the ring is long enough to split into `shards` segments
  // (>= 64 cars each, temporal blocking eligible).
  static bool can_shard(const SimParams& params, unsigned shards);

  void set_state(const uint64_t* x, const uint64_t* v, size_t n) override;
  void set_state32(const uint32_t* x, const uint32_t* v, size_t n) override;
  void advance(uint64_t steps) override;
  void enqueue(uint64_t steps) override;
  void synchronize() override;
  uint64_t steps_done() const override;
  uint64_t checksum() const override;
  const std::vector<Frame>& frames() const override;
  const SimParams& params() const override;
  void observables(double* density, double* mean_velocity, double* flow) override;
  void state(uint64_t* positions, uint64_t* velocities) override;
  void state_segment(uint64_t* positions, uint64_t* velocities, uint64_t* first_rank) override;
  void state_segment32(uint32_t* positions, uint32_t* velocities, uint64_t* first_rank) override;
  void state_segment_async(uint64_t* positions, uint64_t* velocities, uint64_t* first_rank) override;
  void state_wait() override;
  void set_state_segment(const uint64_t* x, const uint64_t* v, size_t n) override;
  size_t sumv_series(uint64_t* out, size_t cap) override;
  size_t wrap_series(uint64_t* out, size_t cap) override;
  void set_checksum(bool enabled) override;
  void* cuda_stream() const override;
  uint64_t kernel_launches() const override;
  int steps_per_launch() const override;
  void shard_range(uint64_t* first, uint64_t* count) const override;
  int exchange_mode() const override;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

// The reference's cell-array engine (NASCH_ENGINE_GRID_REFERENCE,
// src/model.cpp:77-129, src/engine.cpp:186-196) on the GPU (grid.cu).
class GpuGrid : public RingEngine {
 public:
  explicit GpuGrid(const SimParams& params);
  ~GpuGrid() override;

  void set_state(const uint64_t* x, const uint64_t* v, size_t n) override;
  void set_state32(const uint32_t* x, const uint32_t* v, size_t n) override;
  void advance(uint64_t steps) override;
  void enqueue(uint64_t steps) override;
  void synchronize() override;
  uint64_t steps_done() const override;
  uint64_t checksum() const override;
  const std::vector<Frame>& frames() const override;
  const SimParams& params() const override;
  void observables(double* density, double* mean_velocity, double* flow) override;
  void state(uint64_t* positions, uint64_t* velocities) override;
  size_t sumv_series(uint64_t* out, size_t cap) override;
  size_t wrap_series(uint64_t* out, size_t cap) override;
  void set_checksum(bool enabled) override;
  void* cuda_stream() const override;
  uint64_t kernel_launches() const override;
  int steps_per_launch() const override;
  void shard_range(uint64_t* first, uint64_t* count) const override;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

// NCCL unique id (128 bytes) for ShardedRing's distributed constructor;
// rank 0 creates it and the launcher broadcasts it.
void nccl_unique_id(void* out128);

// Extension: seeded uniform distinct sorted positions (selection sampling)
// and velocities uniform in [0, vmax_init] -- the BASELINE.json inputs.
void fill_uniform_state(uint64_t L, uint64_t N, uint64_t vmax_init,
                        uint64_t seed, uint32_t* x, uint32_t* v);

}  // namespace nb200
