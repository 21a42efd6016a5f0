// ensemble.hpp -- many independent rings on one GPU (CUDA-free header).
//
// BASELINE.json config 4 (fundamental diagram: 4096 rings of L=1e5 with
// densities 0.05..0.5, p in {0..0.7}, 8 replica seeds) is a batch of
// independent simulations, each exactly the reference's single-ring model
// (src/model.cpp:42-75) with its own parameters and its own minstd stream
// (src/lcg.cpp:11-16).  The reference would run them one Engine at a time;
// here one launch advances all of them, each ring resident in one SM's
// shared memory for the whole launch.  Multi-GPU: rings shard across ranks
// with no communication.
#pragma once
#include <cstddef>
#include <cstdint>
#include <memory>
#include <vector>

#include "host_model.hpp"

namespace nb200 {

class GpuEnsemble {
 public:
  // One SimParams per ring (output mode and stride are ignored).
  explicit GpuEnsemble(const std::vector<SimParams>& rings);
  ~GpuEnsemble();
  GpuEnsemble(const GpuEnsemble&) = delete;
  GpuEnsemble& operator=(const GpuEnsemble&) = delete;

  size_t size() const;
  // Rank-ordered state of one ring (same validation as GpuRing::set_state).
  void set_state32(size_t ring, const uint32_t* x, const uint32_t* v, size_t n);
  // Every ring at once: rings concatenated in ring order (total = sum of
  // ncars), validated in parallel host chunks, one upload.
  void set_state_all32(const uint32_t* x, const uint32_t* v, size_t total);
  // Advances every ring by min(steps, its remaining steps); synchronous.
  void advance(uint64_t steps);
  void enqueue(uint64_t steps);
  void synchronize();

  uint64_t steps_done(size_t ring);
  // Exact sum over all completed steps of the ring's velocity sum
  // (time-averaged flux = total / (steps * L)).
  void sumv_totals(uint64_t* out, size_t cap);
  // Velocity sum after the last completed step, per ring.
  void sumv_last(uint64_t* out, size_t cap);
  void state(size_t ring, uint64_t* x, uint64_t* v);
  void* cuda_stream() const;
  uint64_t kernel_launches() const;
  size_t resident_capacity_cars() const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

}  // namespace nb200
