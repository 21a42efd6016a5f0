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
#include "tb_config.hpp"

namespace nb200 {

constexpr int kHeadCars = kTbHalo;  // halo depth = the deepest launch (k <= kTbHalo)
constexpr int kConeMax = 256;  // cone slots (one block)
constexpr int kXchgWords = 2 * kHeadCars + 2 * kConeMax;  // u32 per shard record
constexpr uint32_t kFlagWords = 64;  // peer exchange: flag words ahead of the receive slots (max shards)

// Record layout: [0,16) x of local cars 0..15, [16,32) their v,
// [32 + 2i] / [33 + 2i] x / v of cone slot i if this shard owns it.
// Word w of this shard's record for the window at rank offset W.
template <typename VT>
__device__ __forceinline__ uint32_t shard_record_word(const RingArgs& ra, const uint32_t* X, const VT* V,
                                                      uint32_t W, uint32_t w) {
  if (w < 2 * kHeadCars) {
    const uint32_t i = w % kHeadCars;
    return w < kHeadCars ? __ldcg(X + i) : static_cast<uint32_t>(__ldcg(V + i));
  }
  const uint32_t i = (w - 2 * kHeadCars) / 2;
  const uint32_t M = ra.kplan * ra.vmax;
  if (i >= M + ra.kplan) return 0u;
  const uint32_t local = cone_slot_id(ra.n, W, M, i) - ra.gofs;  // wraps when id < gofs
  if (local >= ra.nl) return 0u;
  return (w & 1u) ? static_cast<uint32_t>(__ldcg(V + local)) : __ldcg(X + local);
}

template <typename VT>
__global__ void __launch_bounds__(kConeMax) shard_pack_kernel(const RingArgs ra, uint32_t* send) {
  const Ctl* ctl = ra.ctl;
  const int b = static_cast<int>(ctl->buf);
  const uint32_t* X = xbuf(ra, b);
  const VT* V = vbuf<VT>(ra, b);
  for (uint32_t w = threadIdx.x; w < kXchgWords; w += kConeMax) send[w] = shard_record_word(ra, X, V, ctl->W, w);
}

// ---- peer-memory exchange (kXchgP2P) --------------------------------------
// Every shard h owns a receive area  rec_h[2][G][kXchgWords]  and flags
// flag_h[G].  Launch n of shard g ends (tb_body<PUSH>, its last block) by
// storing its record for the window after the launch into slot
// [seq & 1][g] of EVERY shard -- NVLink stores into peer HBM (pointers from
// cudaIpcOpenMemHandle across processes, or peer access within one) -- and
// then, after a system-scope fence, flag_h[g] = seq.  The plan kernel of
// launch n+1 on shard h waits for flag_h[*] >= seq and reads the slots
// locally.  Two slots suffice: shard g can publish seq+2 only after its own
// plan for seq+1, which needed every shard's seq+1 record, which each shard
// h published only after its plan for seq had finished reading slot
// [seq & 1].  Flags only grow (seq is the ring's launch counter), so they
// are never reset.
struct XchgArgs {
  uint32_t* const* rec = nullptr;   // [G] receive areas, in this process's address space
  uint32_t* const* flag = nullptr;  // [G] flag arrays
  uint32_t g = 0, G = 0, seq = 0;
};

__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// Called by all NT threads of the launch's last block once every block's
// state writes are visible (ticket pattern); W = the rank offset after the
// launch.
template <typename VT, int NT>
__device__ void shard_push(const RingArgs& ra, const uint32_t* X, const VT* V, uint32_t W, const XchgArgs& xa) {
  const size_t slot = (size_t(xa.seq & 1u) * xa.G + xa.g) * kXchgWords;
  for (uint32_t w = threadIdx.x; w < kXchgWords; w += NT) {
    const uint32_t val = shard_record_word(ra, X, V, W, w);
    for (uint32_t h = 0; h < xa.G; ++h) xa.rec[h][slot + w] = val;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < xa.G) st_release_sys_u32(xa.flag[threadIdx.x] + xa.g, xa.seq);
}

// shard_lo[0..G] are the shards' first global ids (shard_lo[G] = N).
// flags != nullptr (peer-memory exchange): first wait until every shard
// has published record `seq` (bounded: ~30 s, then Ctl::err = 3 and no
// plan), then read slot [seq & 1] of recv (= this shard's receive area).
template <typename VT>
__global__ void __launch_bounds__(kConeMax)
    shard_plan_kernel(const RingArgs ra, const uint32_t* recv, const uint32_t* shard_lo, uint32_t G,
                      uint32_t g, const uint32_t* flags, uint32_t seq) {
  Ctl* ctl = ra.ctl;
  const uint32_t i = threadIdx.x;
  if (flags) {
    __shared__ uint32_t s_late;
    if (i == 0) s_late = 0;
    __syncthreads();
    if (i < G) {
      uint64_t t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      for (uint32_t it = 0; static_cast<int32_t>(ld_acquire_sys_u32(flags + i) - seq) < 0; ++it) {
        if (it > 64) __nanosleep(128);
        uint64_t now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (now - t0 > 30000000000ull) {
          atomicExch(&s_late, 1u);
          break;
        }
      }
    }
    __syncthreads();
    if (s_late) {
      if (i == 0) atomicCAS(&ctl->err, 0u, 3u);
      return;
    }
    recv += size_t(seq & 1u) * G * kXchgWords;
  }
  const uint64_t t = ctl->t;
  const uint32_t W = ctl->W;
  const int b = static_cast<int>(ctl->buf);
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
    x = __ldcv(rec + 2 * kHeadCars + 2 * i);
    v = __ldcv(rec + 2 * kHeadCars + 2 * i + 1);
  }
  cone_simulate<kConeMax>(ra, x, v, t, W, kk, ctl);
  if (i < kHeadCars) {  // halo: the next shard's first cars, inline after ours
    const uint32_t* nxt = recv + size_t((g + 1) % G) * kXchgWords;
    xbuf(ra, b)[ra.nl + i] = __ldcv(nxt + i);
    vbuf_w<VT>(ra, b)[ra.nl + i] = static_cast<VT>(__ldcv(nxt + kHeadCars + i));
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
