// dr_kernel.cuh -- distributed-resident step kernel for medium rings
// (4096 < N <= ~600k cars): the whole ring stays in the registers of G
// worker CTAs (one per SM, cooperative launch) for every step of a launch,
// and one planner CTA produces each epoch's origin-cone plan.
//
// A launch runs `steps` steps as epochs of k <= K steps (temporal blocking,
// as nasch_tb_kernel).  Worker g owns the car-id
// segment [seg[g], seg[g+1]) (16-aligned floor partition) plus a 16-car
// halo: the first cars of segment g+1, re-read at every epoch start.  Its
// cars never leave registers between epochs; per epoch it
//   1. waits for plan(e) (epoch 0: the plan in Ctl from the previous launch),
//   2. reloads the halo from the state buffer of epoch e,
//   3. runs k steps (block-wide leader hand-off, one barrier per step),
//   4. stores its owned cars into the buffer of epoch e+1, adds its per-step
//      velocity sums / crossing counts into the step records and signals.
// The planner waits for all G signals of epoch e, checks the counted
// crossings against plan(e), simulates the origin cone from the stored
// state for the next K steps (cone_plan, step_kernels.cuh) and publishes
// plan(e+1).  After the last epoch it plans the next launch into Ctl.
//
// Compared with one TB launch per 16 steps this removes the launch gap, the
// state reload and the end-of-launch ticket per epoch (BASELINE config 2:
// 2e5 cars, where a TB launch is ~10x longer than its arithmetic).
//
// Every wait is bounded: a CTA that waits for more than ~2 s raises
// `abort` and flags Ctl::err = 3, and every other waiter leaves on `abort`,
// so a fault cannot hang the GPU.
#pragma once
#include <cstdint>
#include <type_traits>

#include "step_kernels.cuh"

namespace nb200 {

#ifdef NB_DR_TRACE
// Diagnostic build only: per-epoch %globaltimer stamps (tools/dr_trace.py).
__device__ unsigned long long g_dr_trace[256 * 8];
#define DR_TRACE(e, slot)                                                   \
  do {                                                                      \
    if ((e) < 256) {                                                        \
      unsigned long long tt;                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));                \
      g_dr_trace[(e) * 8 + (slot)] = tt;                                    \
    }                                                                       \
  } while (0)
#else
#define DR_TRACE(e, slot) \
  do {                    \
  } while (0)
#endif

constexpr int kDrTPB = 256;
constexpr uint32_t kDrHalo = 16;

struct DrSync {
  unsigned int done[2];     // workers finished with epoch e (slot e & 1)
  unsigned int plan_epoch;  // plan(e) is published for e <= plan_epoch
  unsigned int abort;
};

struct DrArgs {
  Ctl* plans;              // [2]: plan of epoch e in plans[e & 1] (e >= 1)
  DrSync* sync;            // zeroed before every launch
  const uint32_t* seg;     // [G + 1] segment starts, seg[G] = N
  uint32_t G;              // worker CTAs; block G is the planner
  uint32_t K;              // steps per epoch (the cone plan length)
};

__device__ __forceinline__ unsigned int ld_relaxed_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Thread-0 spin until *p >= target; false when the launch is aborting.
// Polls with relaxed (L2) loads and fences once on success: an acquire load
// per poll would invalidate L1 every iteration.
__device__ __noinline__ bool dr_wait_geq(const unsigned int* p, unsigned int target, DrSync* sync, Ctl* ctl) {
  const long long start = clock64();
  for (uint32_t i = 0;; ++i) {
    if (ld_relaxed_u32(p) >= target) {
      __threadfence();
      return true;
    }
    if ((i & 63u) == 63u) {
      if (ld_relaxed_u32(&sync->abort)) return false;
      if (clock64() - start > 4000000000ll) {  // ~2 s at 1.9 GHz
        atomicExch(&sync->abort, 1u);
        atomicCAS(&ctl->err, 0u, 3u);
        return false;
      }
      if (i > 4096) __nanosleep(64);
    }
  }
}

// Block-wide: thread 0 waits, everyone learns the outcome.
__device__ __forceinline__ bool dr_block_wait(const unsigned int* p, unsigned int target, DrSync* sync,
                                              Ctl* ctl) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) s_ok = dr_wait_geq(p, target, sync, ctl) ? 1 : 0;
  __syncthreads();
  return s_ok != 0;
}

template <typename VT, int TPB>
__device__ void dr_planner(const RingArgs& ra, const DrArgs& da, const uint32_t steps) {
  Ctl* ctl = ra.ctl;
  DrSync* sync = da.sync;
  const uint32_t N = ra.n;
  const uint64_t t0 = ctl->t;
  const int b0 = static_cast<int>(ctl->buf);
  const uint32_t nE = (steps + da.K - 1) / da.K;
  __shared__ uint32_t s_bad, s_Wn;
  for (uint32_t e = 0; e < nE; ++e) {
    const uint32_t k = min(da.K, steps - e * da.K);
    const uint64_t te = t0 + uint64_t(e) * da.K;
    Ctl* pl = e == 0 ? ctl : da.plans + (e & 1u);
    if (!dr_block_wait(&sync->done[e & 1u], da.G, sync, ctl)) return;
    if (threadIdx.x == 0) DR_TRACE(e, 4);
    if (threadIdx.x == 0) {
      sync->done[e & 1u] = 0;  // reused by epoch e + 2, which waits for plan(e + 2)
      s_bad = ~0u;
    }
    __syncthreads();
    // Check the workers' crossing counts against the plan.
    if (threadIdx.x < k) {
      const uint32_t j = threadIdx.x;
      StepRec* r = ra.rec + ((te + j) % kRecCap);
      const uint32_t c = __ldcg(&r->c);
      const uint32_t ck = __ldcg(&pl->ck[j]);
      r->W = __ldcg(&pl->Wk[j]);
      r->cplan = ck;
      if (c != ck) atomicMin(&s_bad, j);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_bad != ~0u && atomicCAS(&ctl->err, 0u, 1u) == 0u) ctl->err_step = static_cast<unsigned int>(te + s_bad);
      uint32_t Wn = __ldcg(&pl->Wk[k - 1]) + __ldcg(&pl->ck[k - 1]);
      if (Wn >= N) Wn -= N;
      s_Wn = Wn;
    }
    __syncthreads();
    const uint32_t Wn = s_Wn;
    const uint64_t tn = te + k;
    const int bn = (b0 + static_cast<int>(e) + 1) & 1;
    const bool last = e + 1 == nE;
    Ctl* dst = last ? ctl : da.plans + ((e + 1) & 1u);
    const uint32_t kk = last ? ra.kplan : da.K;
    if (threadIdx.x == 0) DR_TRACE(e, 5);
    cone_plan<VT, TPB>(ra, xbuf(ra, bn), vbuf<VT>(ra, bn), tn, Wn, kk, dst);
    if (threadIdx.x == 0) DR_TRACE(e, 6);
    for (uint32_t j = threadIdx.x; j < kk; j += TPB) {
      StepRec* r = ra.rec + ((tn + j) % kRecCap);
      r->sumv = 0;
      r->c = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (last) {
        ctl->W = Wn;
        ctl->t = tn;
        ctl->buf = static_cast<unsigned int>(bn);
      } else {
        __threadfence();
        atomicExch(&sync->plan_epoch, e + 1);
        DR_TRACE(e, 7);
      }
    }
  }
}

template <typename VT, int TPB, int CPT>
__global__ void __launch_bounds__(TPB, 1) ring_dr_kernel(const RingArgs ra, const DrArgs da, const uint32_t steps) {
  using Acc = typename std::conditional<sizeof(VT) == 1, uint32_t, unsigned long long>::type;
  constexpr int NW = TPB / 32;
  if (blockIdx.x == da.G) {
    dr_planner<VT, TPB>(ra, da, steps);
    return;
  }
  __shared__ uint32_t s_W[kPlanMax], s_E[kPlanMax], s_E2[kPlanMax];
  __shared__ uint32_t s_lead[2][NW];
  __shared__ Acc s_acc[kPlanMax][TPB];
  Ctl* ctl = ra.ctl;
  DrSync* sync = da.sync;
  const uint32_t N = ra.n, L = ra.L, vmax = ra.vmax, tp = ra.tp;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint64_t t0 = ctl->t;
  const int b0 = static_cast<int>(ctl->buf);
  const uint32_t g = blockIdx.x;
  const uint32_t lo = da.seg[g], S = da.seg[g + 1] - lo;  // owned cars
  const uint32_t span = S + kDrHalo;                     // cars held (owned + halo)
  const uint32_t i0 = threadIdx.x * CPT;
  const uint32_t base = lo + i0;  // id of car 0 (>= N past the ring's end)
  // Car c of this thread holds local index min(i0 + c, span - 1): slots past
  // the halo replicate its front car (their results are never used).
  uint32_t idc[CPT], ap[CPT], x[CPT], v[CPT];
  uint32_t own = 0;
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const uint32_t li = min(i0 + c, span - 1);
    uint32_t id = lo + li;
    const bool wrapped = id >= N;
    if (wrapped) id -= N;
    idc[c] = id;
    uint32_t a = powmod(kA, id);  // once per launch
    ap[c] = a << 1;
    own |= (i0 + c < S) ? (1u << c) : 0u;
  }
  const bool own_all = own == (1u << CPT) - 1u;
  const bool nowrap = base + CPT <= N;  // ids of this thread's cars run consecutively
  const bool active = i0 < span;
  const uint32_t nE = (steps + da.K - 1) / da.K;
  uint32_t phase = 0;
#pragma unroll
  for (int j = 0; j < kPlanMax; ++j) s_acc[j][threadIdx.x] = 0;
  for (uint32_t e = 0; e < nE; ++e) {
    const uint32_t k = min(da.K, steps - e * da.K);
    const uint64_t te = t0 + uint64_t(e) * da.K;
    const int bi = (b0 + static_cast<int>(e)) & 1;
    const Ctl* pl = e == 0 ? ctl : da.plans + (e & 1u);
    if (e > 0 && !dr_block_wait(&sync->plan_epoch, e, sync, ctl)) return;
    if (g == 0 && threadIdx.x == 0) DR_TRACE(e, 0);
    if (threadIdx.x < k) {
      s_W[threadIdx.x] = __ldcg(&pl->Wk[threadIdx.x]);
      s_E[threadIdx.x] = __ldcg(&pl->Ek[threadIdx.x]);
      s_E2[threadIdx.x] = __ldcg(&pl->E2k[threadIdx.x]);
    }
    // (Re)load: everything at the first epoch, the halo afterwards.
    const uint32_t* X = xbuf(ra, bi);
    const VT* V = vbuf<VT>(ra, bi);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if (e == 0 || !((own >> c) & 1u)) {
        x[c] = __ldcg(X + idc[c]);
        v[c] = static_cast<uint32_t>(__ldcg(V + idc[c]));
      }
    }
    __syncthreads();
    uint32_t xmax = x[0];
#pragma unroll
    for (int c = 1; c < CPT; ++c) xmax = max(xmax, x[c]);
    const bool plain = nowrap && xmax < L - k * vmax;
    for (uint32_t j = 0; j < k; ++j) {
      const uint32_t E = s_E[j], E2 = s_E2[j];
      const uint32_t bound = N - s_W[j];
      const uint32_t slot = phase++ & 1u;
      if (lane == 0) s_lead[slot][warp] = x[0];
      __syncthreads();
      uint32_t xn = __shfl_down_sync(0xffffffffu, x[0], 1);
      if (lane == 31) xn = (warp + 1 < NW) ? s_lead[slot][warp + 1] : x[CPT - 1];
      if (!active) continue;
      if (plain && !(base < bound && bound <= base + CPT)) {
        const uint32_t Es = base < bound ? E : E2;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const uint32_t s = mulmod_x2(ap[c], Es);
          const uint32_t xl = (c + 1 < CPT) ? x[c + 1] : xn;
          const uint32_t d = x[c] * ra.neg1 + xl;
          const int vc = static_cast<int>(min(min(v[c] + 1, vmax), d - 1));
          int dec;
          asm("mul.hi.s32 %0, %1, 1;" : "=r"(dec) : "r"(static_cast<int>(s - tp)));
          v[c] = static_cast<uint32_t>(max(vc + dec, 0));
          x[c] += v[c];
        }
        if (own_all) {
          s_acc[j][threadIdx.x] += static_cast<Acc>(VSum<uint32_t, CPT>::sum(v));
        } else if (own) {
          Acc sum = 0;
#pragma unroll
          for (int c = 0; c < CPT; ++c) sum += ((own >> c) & 1u) ? v[c] : 0u;
          s_acc[j][threadIdx.x] += sum;
        }
      } else {
        Acc sum = 0;
        uint32_t crs = 0;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const uint32_t s = mulmod_x2(ap[c], idc[c] < bound ? E : E2);
          const uint32_t xl = (c + 1 < CPT) ? x[c + 1] : xn;
          uint32_t cr = 0;
          v[c] = car_any(x[c], xl, v[c], s, L, vmax, tp, x[c], cr);
          const bool mine = (own >> c) & 1u;
          sum += mine ? v[c] : 0u;
          crs += mine ? cr : 0u;
        }
        s_acc[j][threadIdx.x] += sum;
        if (crs) atomicAdd(&ra.rec[(te + j) % kRecCap].c, crs);
      }
    }
    if (g == 0 && threadIdx.x == 0) DR_TRACE(e, 1);
    // Owned cars into the next epoch's buffer.
    uint32_t* Xo = xbuf(ra, bi ^ 1);
    VT* Vo = vbuf_w<VT>(ra, bi ^ 1);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if ((own >> c) & 1u) {
        Xo[idc[c]] = x[c];
        Vo[idc[c]] = static_cast<VT>(v[c]);
      }
    }
    __syncthreads();
    for (uint32_t j = warp; j < k; j += NW) {
      unsigned long long acc = 0;
#pragma unroll
      for (int q = 0; q < TPB / 32; ++q) acc += s_acc[j][lane + 32 * q];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0 && acc) atomicAdd(&ra.rec[(te + j) % kRecCap].sumv, acc);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPlanMax; ++j) s_acc[j][threadIdx.x] = 0;
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&sync->done[e & 1u], 1u);
      if (g == 0) DR_TRACE(e, 2);
      if (g + 1 == da.G) DR_TRACE(e, 3);
    }
  }
}

}  // namespace nb200
