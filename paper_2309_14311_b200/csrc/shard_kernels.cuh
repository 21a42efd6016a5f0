// shard_kernels.cuh -- the per-launch exchange of the segmented multi-GPU
// ring.
//
// Shard g owns global ids [gofs, gofs + nl) (the make_partition formula of
// src/engine.cpp:31-42) and keeps a 16-car halo -- the first cars of shard
// g+1 -- inline after its own cars.  Before each k-step launch every shard
// needs (a) that halo at step t and (b) the same origin-cone plan.  Each
// shard packs its first 16 cars and the cone slots it owns into a fixed
// record; one all-gather of the records (NCCL across processes, peer copies
// between shards of one process) lets every shard assemble the cone window,
// simulate it redundantly (cone_simulate, identical on every shard) and copy
// its halo.  No other cross-GPU traffic: per-step velocity sums and crossing
// counts stay per shard and are summed on the host.
#pragma once
#include <cstdint>

#include "step_kernels.cuh"

namespace nb200 {

constexpr int kHeadCars = 16;  // halo depth, >= kPlanMax
constexpr int kConeMax = 256;  // cone slots (one block)
constexpr int kXchgWords = 2 * kHeadCars + 2 * kConeMax;  // u32 per shard record

// Record layout: [0,16) x of local cars 0..15, [16,32) their v,
// [32 + 2i] / [33 + 2i] x / v of cone slot i if this shard owns it.
template <typename VT>
__global__ void __launch_bounds__(kConeMax) shard_pack_kernel(const RingArgs ra, uint32_t* send) {
  const Ctl* ctl = ra.ctl;
  const int b = static_cast<int>(ctl->buf);
  const uint32_t* X = xbuf(ra, b);
  const VT* V = vbuf<VT>(ra, b);
  const uint32_t i = threadIdx.x;
  if (i < kHeadCars) {
    send[i] = X[i];
    send[kHeadCars + i] = static_cast<uint32_t>(V[i]);
  }
  const uint32_t M = ra.kplan * ra.vmax;
  uint32_t x = 0, v = 0;
  if (i < M + ra.kplan) {
    const uint32_t id = cone_slot_id(ra.n, ctl->W, M, i);
    const uint32_t local = id - ra.gofs;  // wraps to a huge value when id < gofs
    if (local < ra.nl) {
      x = X[local];
      v = static_cast<uint32_t>(V[local]);
    }
  }
  send[2 * kHeadCars + 2 * i] = x;
  send[2 * kHeadCars + 2 * i + 1] = v;
}

// shard_lo[0..G] are the shards' first global ids (shard_lo[G] = N).
template <typename VT>
__global__ void __launch_bounds__(kConeMax)
    shard_plan_kernel(const RingArgs ra, const uint32_t* recv, const uint32_t* shard_lo, uint32_t G,
                      uint32_t g) {
  Ctl* ctl = ra.ctl;
  const uint64_t t = ctl->t;
  const uint32_t W = ctl->W;
  const int b = static_cast<int>(ctl->buf);
  const uint32_t i = threadIdx.x;
  const uint32_t kk = ra.kplan;
  const uint32_t M = kk * ra.vmax;
  uint32_t x = 0, v = 0;
  if (i < M + kk) {
    const uint32_t id = cone_slot_id(ra.n, W, M, i);
    uint32_t lo = 0, hi = G;  // owner: last shard with shard_lo <= id
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) / 2;
      if (shard_lo[mid] <= id) lo = mid; else hi = mid;
    }
    const uint32_t* rec = recv + size_t(lo) * kXchgWords;
    x = rec[2 * kHeadCars + 2 * i];
    v = rec[2 * kHeadCars + 2 * i + 1];
  }
  cone_simulate<kConeMax>(ra, x, v, t, W, kk, ctl);
  if (i < kHeadCars) {  // halo: the next shard's first cars, inline after ours
    const uint32_t* nxt = recv + size_t((g + 1) % G) * kXchgWords;
    xbuf(ra, b)[ra.nl + i] = nxt[i];
    vbuf_w<VT>(ra, b)[ra.nl + i] = static_cast<VT>(nxt[kHeadCars + i]);
  }
  for (uint32_t j = i; j < kk; j += kConeMax) {
    StepRec* r = ra.rec + ((t + j) % kRecCap);
    r->sumv = 0;
    r->c = 0;
  }
}

// init_state (model.cpp:30-40) for a shard's segment: x = floor(id*L/N).
template <typename VT>
__global__ void shard_init_kernel(uint32_t* x, VT* v, uint32_t nl, uint32_t npad, uint32_t gofs,
                                  uint32_t n, uint64_t L) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < npad;
       i += (uint64_t)gridDim.x * blockDim.x) {
    x[i] = i < nl ? static_cast<uint32_t>((gofs + i) * L / n) : 0u;
    v[i] = 0;
  }
}

}  // namespace nb200
