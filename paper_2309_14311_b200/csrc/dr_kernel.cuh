// dr_kernel.cuh -- distributed-resident step kernel for medium rings
// (4096 < N <= ~600k cars): the whole ring stays in the registers of G
// worker CTAs (one per SM, cooperative launch) for every step of a launch,
// and one planner CTA produces the origin-cone plan of each epoch one epoch
// ahead, off the workers' critical path.
//
// A launch runs `steps` steps as epochs of k <= K steps (temporal blocking,
// as nasch_tb_kernel).  Worker g owns the car-id
// segment [seg[g], seg[g+1]) (16-aligned) plus a 16-car halo: the first
// cars of the next segment, re-read at every epoch start.  Its own cars
// never leave registers; per epoch e it
//   1. waits for plan(e) (epoch 0: the plan in Ctl) and for worker g+1 to
//      have published the state S_e (its flag >= e),
//   2. reloads the halo from S_e's buffer, runs k steps (block-wide leader
//      hand-off, one barrier per step),
//   3. waits until worker g-1 finished epoch e-1 (it has read its halo from
//      the buffer about to be overwritten), stores its cars as S_{e+1}, adds
//      its per-step velocity sums / crossing counts into the step records
//      and raises its flag to e+1.
// The planner, at epoch e, waits until every worker published S_e, checks
// epoch e-1's counted crossings against plan(e-1), simulates the origin cone
// from S_e for k_e + K steps in one warp (cone_warp.cuh) and publishes the
// last K of them as plan(e+1) -- while the workers run epoch e.  After the
// last epoch it installs the next launch's plan in Ctl.
//
// No worker can run more than two epochs ahead of any other (plan(e) needs
// every worker past e-2), which is what makes two plan slots and two state
// buffers enough.  Every wait is bounded: a CTA waiting longer than
// NASCH_B200_DR_TIMEOUT_S (default 60 s, wall time by %globaltimer)
// raises `abort` and Ctl::err = 3, and every other waiter leaves on
// `abort`, so a fault cannot hang the GPU.
#pragma once
#include <cstdint>
#include <type_traits>

#include "cone_warp.cuh"
#include "step_kernels.cuh"

namespace nb200 {

#ifdef NB_DR_TRACE
// Diagnostic build only: per-epoch %globaltimer stamps (tools/dr_trace.py).
__device__ unsigned long long g_dr_trace[256 * 8];
__device__ unsigned long long g_dr_wtrace[64 * 160 * 4];  // [epoch][worker][ready, steps, checked, signalled]
#define DR_TRACE(e, slot)                                                   \
  do {                                                                      \
    if ((e) < 256) {                                                        \
      unsigned long long tt;                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));                \
      g_dr_trace[(e) * 8 + (slot)] = tt;                                    \
    }                                                                       \
  } while (0)
#define DR_WTRACE(e, g, slot)                                              \
  do {                                                                      \
    if ((e) < 64 && (g) < 160) {                                            \
      unsigned long long tt;                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));                \
      g_dr_wtrace[((e) * 160 + (g)) * 4 + (slot)] = tt;                     \
    }                                                                       \
  } while (0)
#else
#define DR_WTRACE(e, g, slot) \
  do {                        \
  } while (0)
#define DR_TRACE(e, slot) \
  do {                    \
  } while (0)
#endif

constexpr int kDrTPB = 256;
constexpr uint32_t kDrHalo = 32;  // >= K (epochs of up to 32 steps)
constexpr uint32_t kDrKMax = 32;

struct DrSync {
  unsigned int plan_epoch;  // plan(e) is published for e <= plan_epoch
  unsigned int abort;
  unsigned int flags[1];    // [G]: epochs worker g has finished (S_flag published)
};

struct DrArgs {
  Ctl* plans;              // [2]: plan of epoch e in plans[e & 1] (e >= 1)
  uint32_t* mbox;          // [3][G][2 * kDrHalo]: worker g's first cars (x, v) of S_e in slot e % 3
  DrSync* sync;            // zeroed before every launch (2 + G words)
  const uint32_t* seg;     // [G + 1] segment starts, seg[G] = N
  uint32_t G;              // worker CTAs; block G is the planner
  uint32_t K;              // steps per epoch (the cone plan length)
};

__device__ __forceinline__ unsigned int ld_relaxed_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Bound on any single wait, in %globaltimer nanoseconds (wall time, so it
// does not depend on the SM clock): NASCH_B200_DR_TIMEOUT_S, default 60 s
// (engine.cu).  A wait that long means a worker CTA is not running (a
// time-sliced or preempted GPU, a debugger); the launch then aborts with
// Ctl::err = 3, reported at the next drain.
static __constant__ unsigned long long c_dr_timeout_ns = 60ull * 1000000000ull;

__device__ __forceinline__ unsigned long long dr_now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Thread-0 spin until *p >= target; false when the launch is aborting.
// Polls with relaxed (L2) loads and fences once on success: an acquire load
// per poll would invalidate L1 every iteration.
__device__ __noinline__ bool dr_wait_geq(const unsigned int* p, unsigned int target, DrSync* sync, Ctl* ctl) {
  const unsigned long long start = dr_now_ns();
  for (uint32_t i = 0;; ++i) {
    if (ld_relaxed_u32(p) >= target) {
      __threadfence();
      return true;
    }
    if ((i & 63u) == 63u) {
      if (ld_relaxed_u32(&sync->abort)) return false;
      if (dr_now_ns() - start > c_dr_timeout_ns) {
        atomicExch(&sync->abort, 1u);
        atomicCAS(&ctl->err, 0u, 3u);
        return false;
      }
      if (i > 4096) __nanosleep(64);
    }
  }
}

// Publish a flag after this CTA's writes (ordered by the caller's
// __syncthreads): gpu-scope fence, then a plain relaxed store -- no atomic
// round trip.
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  __threadfence();
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// Thread-0 spin until *p >= a and *q >= b (one acquire fence at the end).
__device__ __noinline__ bool dr_wait2(const unsigned int* p, unsigned int a, const unsigned int* q, unsigned int b,
                                      DrSync* sync, Ctl* ctl) {
  const unsigned long long start = dr_now_ns();
  for (uint32_t i = 0;; ++i) {
    const unsigned int vp = ld_relaxed_u32(p), vq = ld_relaxed_u32(q);
    if (vp >= a && vq >= b) {
      __threadfence();
      return true;
    }
    if ((i & 63u) == 63u) {
      if (ld_relaxed_u32(&sync->abort)) return false;
      if (dr_now_ns() - start > c_dr_timeout_ns) {
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

// Block-wide: until every worker's flag is >= target.
__device__ __noinline__ bool dr_wait_all(const DrSync* sync, uint32_t G, unsigned int target, Ctl* ctl) {
  const unsigned long long start = dr_now_ns();
  for (uint32_t i = 0;; ++i) {
    bool ok = true;
    for (uint32_t g = threadIdx.x; g < G; g += blockDim.x) ok = ok && ld_relaxed_u32(&sync->flags[g]) >= target;
    if (__syncthreads_and(ok)) break;
    if ((i & 63u) == 63u) {
      int bad = 0;
      if (threadIdx.x == 0) {
        bad = ld_relaxed_u32(&sync->abort) != 0;
        if (!bad && dr_now_ns() - start > c_dr_timeout_ns) {
          atomicExch(const_cast<unsigned int*>(&sync->abort), 1u);
          atomicCAS(&ctl->err, 0u, 3u);
          bad = 1;
        }
      }
      if (__syncthreads_or(bad)) return false;
    }
  }
  __threadfence();
  return true;
}

// Crossing counts of the k steps from te (all workers done) against plan
// pl; thread j (= threadIdx.x - first) checks step j.
__device__ __forceinline__ void dr_verify(const RingArgs& ra, const Ctl* pl, uint64_t te, uint32_t k, Ctl* ctl,
                                          uint32_t first = 0) {
  if (threadIdx.x >= first && threadIdx.x - first < k) {
    const uint32_t j = threadIdx.x - first;
    StepRec* r = ra.rec + ((te + j) % kRecCap);
    const uint32_t c = __ldcg(&r->c);
    const uint32_t ck = __ldcg(&pl->ck[j]);
    r->W = __ldcg(&pl->Wk[j]);
    r->cplan = ck;
    if (c != ck && atomicCAS(&ctl->err, 0u, 1u) == 0u) ctl->err_step = static_cast<unsigned int>(te + j);
  }
}

template <typename VT, int TPB>
__device__ void dr_planner(const RingArgs& ra, const DrArgs& da, const uint32_t steps) {
  static_assert(TPB >= kConeMwThreads + 32, "cone warps plus verification warps");
  __shared__ ConeTab s_tab;
  __shared__ Ctl s_out;  // the cone's plan, copied out once plan(e-1) was checked
  Ctl* ctl = ra.ctl;
  DrSync* sync = da.sync;
  const uint64_t t0 = ctl->t;
  const int b0 = static_cast<int>(ctl->buf);
  const uint32_t K = da.K;
  const uint32_t nE = (steps + K - 1) / K;
  cone_tab_fill(s_tab, ra);
  __shared__ uint32_t s_W;
  if (threadIdx.x == 0) s_W = ctl->W;
  __syncthreads();
  uint32_t We = s_W;  // rank offset at the start of epoch e
  for (uint32_t e = 0; e < nE; ++e) {
    const uint32_t k = min(K, steps - e * K);
    const uint64_t te = t0 + uint64_t(e) * K;
    // S_e complete, hence every worker is past epoch e-1 and done reading
    // plan(e-1), whose slot receives plan(e+1).
    if (e > 0 && !dr_wait_all(sync, da.G, e, ctl)) return;
    if (threadIdx.x == 0) DR_TRACE(e, 4);
    const int be = (b0 + static_cast<int>(e)) & 1;
    Ctl* dst = da.plans + ((e + 1) & 1u);  // plan(e-1)'s slot
    uint32_t Wn = 0;
    if (threadIdx.x < kConeMwThreads) {
      Wn = cone_mw<VT>(ra, xbuf(ra, be), vbuf<VT>(ra, be), te, We, k + K, k, K, &s_out, s_tab);
    } else if (e > 0) {
      // meanwhile the other warps check epoch e-1 against plan(e-1), which
      // dst still holds
      dr_verify(ra, e == 1 ? ctl : dst, te - K, K, ctl, kConeMwThreads);
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < K; j += TPB) {
      dst->Wk[j] = s_out.Wk[j];
      dst->Ek[j] = s_out.Ek[j];
      dst->E2k[j] = s_out.E2k[j];
      dst->ck[j] = s_out.ck[j];
    }
    if (threadIdx.x == 0) {
      dst->kplan = s_out.kplan;
      dst->E = s_out.E;
      dst->E2 = s_out.E2;
    }
    const uint64_t tn = te + k;
    for (uint32_t j = threadIdx.x; j < K; j += TPB) {
      StepRec* r = ra.rec + ((tn + j) % kRecCap);
      r->sumv = 0;
      r->c = 0;
    }
    if (threadIdx.x == 0) {
      s_W = Wn;
      DR_TRACE(e, 5);
    }
    __syncthreads();
    We = s_W;
    if (threadIdx.x == 0 && e + 1 < nE) {
      st_release_u32(&sync->plan_epoch, e + 1);
      DR_TRACE(e, 7);
    }
  }
  // Last epoch done everywhere: check it, install the next launch's plan.
  if (!dr_wait_all(sync, da.G, nE, ctl)) return;
  const uint32_t kl = steps - (nE - 1) * K;
  dr_verify(ra, nE == 1 ? ctl : da.plans + ((nE - 1) & 1u), t0 + uint64_t(nE - 1) * K, kl, ctl);
  __syncthreads();
  const Ctl* np = da.plans + (nE & 1u);
  if (threadIdx.x < K) {
    ctl->Wk[threadIdx.x] = __ldcg(&np->Wk[threadIdx.x]);
    ctl->Ek[threadIdx.x] = __ldcg(&np->Ek[threadIdx.x]);
    ctl->E2k[threadIdx.x] = __ldcg(&np->E2k[threadIdx.x]);
    ctl->ck[threadIdx.x] = __ldcg(&np->ck[threadIdx.x]);
  }
  if (threadIdx.x == 0) {
    ctl->kplan = K;
    ctl->E = __ldcg(&np->E);
    ctl->E2 = __ldcg(&np->E2);
    ctl->W = We;
    ctl->t = t0 + steps;
    ctl->buf = static_cast<unsigned int>((b0 + static_cast<int>(nE)) & 1);
  }
}

// Cars a worker CTA can hold: NW warp tiles of 32*CPT cars, each with its
// own 16-car halo (the next warp's first cars, or the next segment's).
template <int TPB, int CPT>
constexpr uint32_t dr_capacity() {
  return (TPB / 32) * (32u * CPT - kDrHalo);
}

// QDRAW: the draw of car c of a thread as (E a^id0) a^c -- one product per
// thread and step times the constant-bank 2 a^c, as in nasch_tb_kernel --
// instead of a per-car multiplier register pair and id (three registers per
// car): what lets 32 cars per thread fit, i.e. rings up to ~1.17M cars.
template <typename VT, int TPB, int CPT, bool QDRAW = false>
__global__ void __launch_bounds__(TPB, 1) ring_dr_kernel(const RingArgs ra, const DrArgs da, const uint32_t steps) {
  using Acc = typename std::conditional<sizeof(VT) == 1, uint32_t, unsigned long long>::type;
  constexpr int NW = TPB / 32;
  constexpr uint32_t OW = 32u * CPT - kDrHalo;  // cars owned per warp tile
  if (blockIdx.x == da.G) {
    dr_planner<VT, TPB>(ra, da, steps);
    return;
  }
  __shared__ uint32_t s_W[kPlanCap], s_E[kPlanCap], s_E2[kPlanCap], s_ck[kPlanCap];
  __shared__ uint32_t s_head[NW][2 * kDrHalo];  // each warp tile's first cars, for the warp behind
  __shared__ Acc s_wacc[kDrKMax][NW];  // per-warp, per-step velocity sums
  Ctl* ctl = ra.ctl;
  DrSync* sync = da.sync;
  const uint32_t N = ra.n, L = ra.L, vmax = ra.vmax, tp = ra.tp;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint64_t t0 = ctl->t;
  const int b0 = static_cast<int>(ctl->buf);
  const uint32_t g = blockIdx.x;
  const uint32_t lo = da.seg[g], S = da.seg[g + 1] - lo;  // owned cars
  const uint32_t wbase = warp * OW;                      // first car of this warp tile
  const bool wactive = wbase < S;                        // warp-uniform
  const uint32_t u0 = lane * CPT;                        // first car within the warp tile
  const uint32_t i0 = wbase + u0;                        // ... within the segment
  const uint32_t base = lo + i0;                         // its id (>= N past the ring's end)
  // Cars past S are the halo (the next segment's first cars; slots past
  // those replicate the last one and are never used).
  const uint32_t span = S + kDrHalo;
  constexpr int NM = QDRAW ? 1 : CPT;  // per-car multipliers and ids only without QDRAW
  uint32_t idc[NM], ap[NM], apB[NM], x[CPT], v[CPT];
  uint32_t own = 0;
  uint32_t P2 = 0;  // QDRAW: 2 a^base
  if constexpr (QDRAW) {
    P2 = (wactive ? powmod(kA, base) : 1u) << 1;  // once per launch
#pragma unroll
    for (int c = 0; c < CPT; ++c) own |= (u0 + c < OW && i0 + c < S) ? (1u << c) : 0u;
  } else {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const uint32_t li = min(i0 + c, span - 1);
      uint32_t id = lo + li;
      const bool wrapped = id >= N;
      if (wrapped) id -= N;
      idc[c] = id;
      uint32_t a = wactive ? powmod(kA, id) : 1u;  // once per launch
      ap[c] = a << 1;                              // ids below the rank seam
      apB[c] = mulmod(a, ra.an_inv) << 1;          // at or past it
      own |= (u0 + c < OW && i0 + c < S) ? (1u << c) : 0u;
    }
  }
  // the id of slot c (halo slots past the span replicate its last car)
  auto slot_id = [&](int c) {
    if constexpr (QDRAW) {
      uint32_t id = lo + min(i0 + static_cast<uint32_t>(c), span - 1);
      if (id >= N) id -= N;
      return id;
    } else {
      return idc[c];
    }
  };
  const bool own_all = CPT == 32 ? own == 0xffffffffu : own == (1u << (CPT & 31)) - 1u;
  const bool nowrap = base + CPT <= N;  // ids of this thread's cars run consecutively
  const uint32_t nE = (steps + da.K - 1) / da.K;
  for (uint32_t i = threadIdx.x; i < kDrKMax * NW; i += TPB) (&s_wacc[0][0])[i] = 0;
  for (uint32_t e = 0; e < nE; ++e) {
    const uint32_t k = min(da.K, steps - e * da.K);
    const uint64_t te = t0 + uint64_t(e) * da.K;
    const int bi = (b0 + static_cast<int>(e)) & 1;
    const Ctl* pl = e == 0 ? ctl : da.plans + (e & 1u);
    // plan(e) published, and the halo's owner has published S_e
    __shared__ int s_ok;
    if (threadIdx.x == 0)
      s_ok = e == 0 || dr_wait2(&sync->plan_epoch, e, &sync->flags[g + 1 == da.G ? 0 : g + 1], e, sync, ctl);
    __syncthreads();
    if (!s_ok) return;
    if (g == 0 && threadIdx.x == 0) DR_TRACE(e, 0);
    if (threadIdx.x == 0) DR_WTRACE(e, g, 0);
    if (threadIdx.x < k) {
      s_W[threadIdx.x] = __ldcg(&pl->Wk[threadIdx.x]);
      s_E[threadIdx.x] = __ldcg(&pl->Ek[threadIdx.x]);
      s_E2[threadIdx.x] = __ldcg(&pl->E2k[threadIdx.x]);
      s_ck[threadIdx.x] = __ldcg(&pl->ck[threadIdx.x]);
    }
    if (e == 0) {  // the whole segment and halo from the state buffer
      const uint32_t* X = xbuf(ra, bi);
      const VT* V = vbuf<VT>(ra, bi);
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const uint32_t id = slot_id(c);
        x[c] = __ldcg(X + id);
        v[c] = static_cast<uint32_t>(__ldcg(V + id));
      }
    } else {
      // Halo slots: the next warp's first cars (shared memory, written at
      // the end of the previous epoch) or worker g+1's mailbox.
      const uint32_t* mb = da.mbox + ((e % 3u) * da.G + (g + 1 == da.G ? 0 : g + 1)) * (2 * kDrHalo);
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        if (!((own >> c) & 1u)) {
          const uint32_t li = min(i0 + c, span - 1);
          if (li < S) {
            const uint32_t h = li - (wbase + OW);  // < kDrHalo: in warp + 1's head
            x[c] = s_head[warp + 1][h];
            v[c] = s_head[warp + 1][kDrHalo + h];
          } else {
            const uint32_t h = li - S;
            x[c] = __ldcg(mb + h);
            v[c] = __ldcg(mb + kDrHalo + h);
          }
        }
      }
    }
    __syncthreads();
    uint32_t xmax = x[0];
#pragma unroll
    for (int c = 1; c < CPT; ++c) xmax = max(xmax, x[c]);
    const bool plain = nowrap && xmax < L - k * vmax;
    if (wactive) {
      // Warp tiles: no block barrier inside the epoch.
      for (uint32_t j = 0; j < k; ++j) {
        const uint32_t E = s_E[j], E2 = s_E2[j];
        const uint32_t bound = N - s_W[j];
        uint32_t xn = __shfl_down_sync(0xffffffffu, x[0], 1);
        if (lane == 31) xn = x[CPT - 1];  // the tile front's leader is unknown: k <= halo
        // Warp-uniform path choice: a lane near the origin or on the rank
        // seam sends the whole warp down the general path (a few more
        // instructions per car) instead of the warp running both.
        const bool tplain = plain && !(base < bound && bound <= base + CPT);
        if (__all_sync(0xffffffffu, tplain)) {
          const uint32_t Es = base < bound ? E : E2;
          const uint32_t Qs = QDRAW ? mulmod_x2(P2, Es) : 0u;
#pragma unroll
          for (int c = 0; c < CPT; ++c) {
            const uint32_t s = QDRAW ? mulmod_x2(c_apow2.v[c], Qs) : mulmod_x2(ap[QDRAW ? 0 : c], Es);
            const uint32_t xl = (c + 1 < CPT) ? x[c + 1] : xn;
            const uint32_t d = x[c] * ra.neg1 + xl;
            const int vc = static_cast<int>(min(min(v[c] + 1, vmax), d - 1));
            int dec;
            asm("mul.hi.s32 %0, %1, 1;" : "=r"(dec) : "r"(static_cast<int>(s - tp)));
            v[c] = static_cast<uint32_t>(max(vc + dec, 0));
            x[c] += v[c];
          }
          uint32_t sum = 0;
          if (own_all) {
            sum = VSum<uint32_t, CPT>::sum(v);
          } else if (own) {
#pragma unroll
            for (int c = 0; c < CPT; ++c) sum += ((own >> c) & 1u) ? v[c] : 0u;
          }
          sum = __reduce_add_sync(0xffffffffu, sum);
          if (lane == 0) s_wacc[j][warp] = sum;
        } else {
          // Any car: seam side per car (precomputed multipliers), headway
          // and position modulo L as unsigned min's (L < 2^31).
          Acc sum = 0;
          uint32_t crs = 0;
          // QDRAW: base E or E2 by rank side, a^-N for ids wrapped past N-1
          const uint32_t QE = QDRAW ? mulmod_x2(P2, E) : 0u, QE2 = QDRAW ? mulmod_x2(P2, E2) : 0u;
          const uint32_t QEw = QDRAW ? mulmod_d(QE, ra.an_inv) : 0u, QE2w = QDRAW ? mulmod_d(QE2, ra.an_inv) : 0u;
#pragma unroll
          for (int c = 0; c < CPT; ++c) {
            uint32_t s;
            if constexpr (QDRAW) {
              const bool wrapped = base + c >= N;
              const uint32_t id = wrapped ? base + c - N : base + c;
              s = mulmod_x2(c_apow2.v[c], id < bound ? (wrapped ? QEw : QE) : (wrapped ? QE2w : QE2));
            } else {
              s = mulmod_x2(idc[c] < bound ? ap[c] : apB[c], E);
            }
            const uint32_t xl = (c + 1 < CPT) ? x[c + 1] : xn;
            uint32_t d = x[c] * ra.neg1 + xl;
            d = min(d, d + L);  // leader past the origin: + L
            const int vc = static_cast<int>(min(min(v[c] + 1, vmax), d - 1));
            int dec;
            asm("mul.hi.s32 %0, %1, 1;" : "=r"(dec) : "r"(static_cast<int>(s - tp)));
            v[c] = static_cast<uint32_t>(max(vc + dec, 0));
            const uint32_t xs = x[c] + v[c];
            x[c] = min(xs, xs - L);
            const bool mine = (own >> c) & 1u;
            sum += mine ? v[c] : 0u;
            crs += (mine && xs >= L) ? 1u : 0u;
          }
          const uint32_t ws = __reduce_add_sync(0xffffffffu, static_cast<uint32_t>(sum));
          if (lane == 0) s_wacc[j][warp] = ws;
          crs = __reduce_add_sync(0xffffffffu, crs);
          if (lane == 0 && crs) atomicAdd(&ra.rec[(te + j) % kRecCap].c, crs);
        }
      }
    }
    if (g == 0 && threadIdx.x == 0) DR_TRACE(e, 1);
    if (threadIdx.x == 0) DR_WTRACE(e, g, 1);
    // S_{e+1}: each warp tile's first cars to shared memory (the halo of the
    // warp behind); the segment's first cars also into mailbox slot
    // (e+1) % 3 (last read as the halo of epoch e-2, which every worker has
    // finished: we hold plan(e)).
    {
      uint32_t* mb = da.mbox + (((e + 1) % 3u) * da.G + g) * (2 * kDrHalo);
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        if (u0 + c < kDrHalo && i0 + c < S) {
          s_head[warp][u0 + c] = x[c];
          s_head[warp][kDrHalo + u0 + c] = v[c];
          if (warp == 0) {
            mb[u0 + c] = x[c];
            mb[kDrHalo + u0 + c] = v[c];
          }
        }
      }
    }
    if (threadIdx.x == 0) DR_WTRACE(e, g, 2);
    // The whole segment into the state buffer only where the planner will
    // read it (the origin cone of S_{e+1}) and at the end of the launch.
    // Readers of that buffer's previous contents (S_{e-1}: the planner's
    // cone at epoch e-1) are done -- plan(e) is out.
    {
      uint32_t Wn = s_W[k - 1] + s_ck[k - 1];
      if (Wn >= N) Wn -= N;
      const uint32_t span_c = 2u * da.K * (vmax + 1);        // cone slots, upper bound
      const uint32_t c0 = cone_slot_id(N, Wn, 2u * da.K * vmax, 0);  // first cone id
      const uint32_t rel = lo >= c0 ? lo - c0 : lo + N - c0;        // segment start past c0
      const bool cone = rel < span_c || rel + S > N;               // ranges intersect (mod N)
      if (e + 1 == nE || cone) {
        uint32_t* Xo = xbuf(ra, bi ^ 1);
        VT* Vo = vbuf_w<VT>(ra, bi ^ 1);
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          if ((own >> c) & 1u) {
            const uint32_t id = slot_id(c);
            Xo[id] = x[c];
            Vo[id] = static_cast<VT>(v[c]);
          }
        }
      }
    }
    __syncthreads();
    if (threadIdx.x < k) {
      unsigned long long acc = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) acc += s_wacc[threadIdx.x][w];
      if (acc) atomicAdd(&ra.rec[(te + threadIdx.x) % kRecCap].sumv, acc);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      st_release_u32(&sync->flags[g], e + 1);
      if (g == 0) DR_TRACE(e, 2);
      DR_WTRACE(e, g, 3);
      if (g + 1 == da.G) DR_TRACE(e, 3);
    }
  }
}

}  // namespace nb200
