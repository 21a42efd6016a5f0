// tb_kernel.cuh -- temporal-blocked NaSch step kernel (k <= 16 steps per
// launch).  See step_kernels.cuh for the shared reformulation (ID order,
// counter-based draws, integer threshold) and DESIGN.md section 4.1.
//
// Tiles of consecutive cars (owned + a HALO of cars ahead) are held in
// registers (CPT cars per thread) for all k steps.  Warp tiles (WT, the
// default for large rings): each warp owns 32*CPT - HALO cars with its own
// halo and passes leaders by shuffle only -- no barrier inside the launch.
// Block tiles (medium rings): one halo per block, one __syncthreads per
// step hands each warp's first position to the warp behind it.  Per step a
// thread takes one of two paths:
//   plain  -- its cars cannot reach the origin within the launch
//             (max x < L - k*vmax at tile start) and the rank seam is not at
//             or inside its cars: gap = leader - x - 1, no mod L, no crossing
//             bookkeeping, one draw base.  This is every thread but a handful
//             near the origin.
//   general-- per-car seam/wrap handling (car_any) and an exact crossing
//             count, added straight to the step's record.
// Exact per-step velocity sums are kept per thread in shared memory (one
// writer per slot, no atomics) and reduced once per launch.  The launch's
// last block verifies the counted crossings against the origin-cone plan and
// plans the next launch (cone_plan, step_kernels.cuh).
#pragma once
#include <cstdint>
#include <type_traits>

#include "shard_kernels.cuh"
#include "step_kernels.cuh"
#include "tb_config.hpp"

namespace nb200 {

// The next launch's origin cone (kplan (vmax + 1) cars, one per thread) is
// simulated by the launch's last block when it fits the block; otherwise
// by cone_init_kernel<VT, 256> enqueued after the launch (engine.cu).
__host__ __device__ __forceinline__ bool tb_plan_inline(uint32_t kplan, uint32_t vmax, int tpb) {
  return kplan * (vmax + 1) <= uint32_t(tpb) && tpb >= 64;
}

#ifdef NB_TB_TRACE
// Experiment builds only: %globaltimer per launch (slot = launch index mod
// 64): [0] first block start, [1] last block start, [2] first block end,
// [3] last block end (before the ticket), [4] plan start, [5] plan end.
static __device__ unsigned long long g_tb_trace[64][8];  // per translation unit
__device__ __forceinline__ unsigned long long tb_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

// A launch over a range of tiles (the streamed end-to-end job, engine.cu
// GpuRing::job32): tiles [tile0, tile_end) with P starting at
// a^(tile0 * STORE) and advancing by gpow = a^(gridDim.x * STORE) per
// grid-stride tile; only the range launch with epi != 0 (the last) runs the
// launch epilogue (plan check, W / t / buf update) -- the earlier ones only
// add their tiles' velocity sums and crossings to the step records.
struct TbRange {
  uint32_t tile0, tile_end, gpow, a_tile0, epi;
};

// The launch body.  PUSH (segmented ring, peer-memory exchange only): the
// launch's last block also publishes this segment's exchange record for the
// next launch straight into every segment's receive slots (shard_push,
// shard_kernels.cuh) -- the pack and the all-gather fused into the step
// kernel.  PUSH = false compiles to the plain kernel (dead code removed).
template <typename VT, int TPB, int CPT, int HALO, bool WT, bool PUSH, bool RANGE = false>
__device__ __forceinline__ void tb_body(const RingArgs& ra, const uint32_t k, const XchgArgs& xa,
                                        const TbRange& rg = TbRange{}) {
  using G = TbGeom<TPB, CPT, HALO, WT>;
  constexpr uint32_t LOAD = G::kLoad;     // cars spanned per block tile
  constexpr uint32_t STORE = G::kStore;   // cars owned (stored) per block tile
  constexpr uint32_t WSTORE = G::kWarpStore;  // owned per halo unit (warp or block)
  constexpr int NW = TPB / 32;
  static_assert(HALO % 16 == 0 && HALO <= kPlanMax && CPT <= 64, "halo bounds the plan; k <= HALO");
  using Acc = typename std::conditional<sizeof(VT) == 1, uint32_t, unsigned long long>::type;
  // per step j: {E, E2, id of the rank-0 car (N - W, N when W = 0), 0}
  __shared__ uint4 s_plan[kPlanMax];
  __shared__ uint32_t s_lead[2][NW];
  __shared__ Acc s_acc[kPlanMax][TPB];  // per-thread, per-step velocity sums

  Ctl* ctl = ra.ctl;
  const uint32_t N = ra.n, L = ra.L, vmax = ra.vmax, tp = ra.tp;
  const uint64_t t = ctl->t;
  const int b = static_cast<int>(ctl->buf);
#ifdef NB_TB_TRACE
  unsigned long long* trc = g_tb_trace[(t / (k ? k : 1)) % 64];
  if (threadIdx.x == 0) {
    const unsigned long long now = tb_now();
    atomicMin(trc + 0, now);
    atomicMax(trc + 1, now);
  }
#endif
  if (threadIdx.x < k) s_plan[threadIdx.x] = make_uint4(ctl->Ek[threadIdx.x], ctl->E2k[threadIdx.x],
                                                        N - ctl->Wk[threadIdx.x], 0u);
  for (uint32_t j = 0; j < k; ++j) s_acc[j][threadIdx.x] = 0;
  __syncthreads();
  const uint32_t* __restrict__ X = xbuf(ra, b);
  const VT* __restrict__ V = vbuf<VT>(ra, b);
  uint32_t* __restrict__ Xo = xbuf(ra, b ^ 1);
  VT* __restrict__ Vo = vbuf_w<VT>(ra, b ^ 1);
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t i0 = G::offset(threadIdx.x);  // first car of this thread within the tile
  // index of car 0 within its halo unit (the warp's tile, or the block's)
  const uint32_t u0 = WT ? lane * CPT : i0;
  const uint32_t reach = k * vmax;        // farthest any car moves in this launch (< L)

  // P = a^(global id of this thread's first car in its first tile).  The
  // draw of car c at step j is E_j a^(id_0 + c) = (E_j P) a^c: one mulmod
  // per thread and step for Q = E_j P, then one per car with the constant
  // 2 a^c as a constant-bank operand (no per-car multiplier registers).
  uint32_t P = mulmod_d(mulmod_d(ra.agofs, __ldg(ra.blkpow + blockIdx.x)), __ldg(ra.thrpow + threadIdx.x));
  if (RANGE) P = mulmod_d(P, rg.a_tile0);
  const uint32_t gpow = RANGE ? rg.gpow : ra.g;
  uint32_t phase = 0;  // running step counter across tiles: s_lead slot parity
  const uint32_t nl = ra.nl;  // cars stored here (a shard's segment, or the ring)
  const uint32_t ntiles = RANGE ? min((nl + STORE - 1) / STORE, rg.tile_end) : (nl + STORE - 1) / STORE;
  for (uint32_t tile = (RANGE ? rg.tile0 : 0u) + blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t a0 = tile * STORE;          // local index of the tile
    const uint32_t bl = a0 + i0;               // local index of car 0
    const uint32_t base = ra.gofs + bl;        // global id of car 0 (may exceed N at the wrap)
    const bool nowrap = ra.gofs + a0 + LOAD <= N;  // block-uniform: ids do not wrap
    // Contiguous in memory: always for a shard (its halo sits inline after
    // nl); on one GPU unless the tile wraps past id N-1.
    const bool fast = ra.sharded || nowrap;
    uint32_t x[CPT], v[CPT];
    if (fast) {
#pragma unroll
      for (int q = 0; q < CPT / 4; ++q) {
        const uint4 r = ld_nc_v4(X + bl + 4 * q);
        x[4 * q] = r.x;
        x[4 * q + 1] = r.y;
        x[4 * q + 2] = r.z;
        x[4 * q + 3] = r.w;
      }
      VLanes<VT, CPT>::load(V + bl, v);
    } else {  // one GPU, wrap tile: ids past N-1 continue at 0
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        uint32_t id = base + c;
        if (id >= N) id -= N;
        x[c] = X[id];
        v[c] = V[id];
      }
    }
#if NB_TB_PREFETCH
    // The warp's cars of its NEXT tile to L2 while this one steps.
    if (WT && lane == 0 && tile + gridDim.x < ntiles) {
      const uint32_t nb = (tile + gridDim.x) * STORE + warp * WSTORE;
      if (ra.gofs + nb + 32u * CPT <= N || ra.sharded) {
        prefetch_l2_bulk(X + nb, 32u * CPT * 4u);
        prefetch_l2_bulk(V + nb, 32u * CPT * sizeof(VT));
      }
    }
#endif
    const uint32_t P2 = P << 1;
    P = mulmod_d(P, gpow);
    // bit c: car c is stored by this tile (all of them but in the halo and
    // at a shard's end)
    const bool own_all = u0 + CPT <= WSTORE && bl + CPT <= nl;
    unsigned long long own = own_all ? ~0ull : 0ull;
    if (!own_all) {
      own = 0ull;
#pragma unroll
      for (int c = 0; c < CPT; ++c) own |= (u0 + c < WSTORE && bl + c < nl) ? (1ull << c) : 0ull;
    }
    uint32_t xmax = x[0];
#pragma unroll
    for (int c = 1; c < CPT; ++c) xmax = max(xmax, x[c]);
    const bool plain = nowrap && xmax < L - reach;
#if NB_TB_MN3
    // Offset form x[c] = position - c (mod 2^32) for the whole tile: the
    // headway IMAD then yields the gap x_{c+1} - x_c - 1 directly.
    // (Measured against a form that also keeps velocity + 1 and position -
    // c + j, so that min(v+1, vmax, gap) needs no add and the clamp is one
    // VIADDMNMX: 9 % fewer instructions per step but 1.7 % slower on C3,
    // round 2.)
#pragma unroll
    for (int c = 1; c < CPT; ++c) x[c] -= c;
#endif
    // Relative form (warp tiles whose cars are all plain): positions minus
    // the warp's first car's, all below 2^24 for the whole launch, so the
    // FP32 add of two bit patterns is their exact integer sum.
    bool frel = false;
    uint32_t xb = 0;
#if NB_TB_FREL && NB_TB_MN3
    if (WT) {
      xb = __shfl_sync(0xffffffffu, x[0], 0);
      const uint32_t xtop = __shfl_sync(0xffffffffu, x[CPT - 1], 31);
      frel = __all_sync(0xffffffffu, plain) && xtop - xb < (1u << 24) - reach - 2u * CPT - vmax - 64u;
      if (frel) {
#pragma unroll
        for (int c = 0; c < CPT; ++c) x[c] -= xb;
      }
    }
#endif

    for (uint32_t j = 0; j < k; ++j) {
      const uint4 pl = s_plan[j];
      const uint32_t E = pl.x, E2 = pl.y, bound = pl.z;
      // Slots alternate with the running step count, so one barrier per step
      // suffices (a slot is rewritten only after the next barrier).
      uint32_t xn;
      if (WT) {
        xn = __shfl_down_sync(0xffffffffu, x[0], 1);
        // warp tiles: the front car of the warp's halo has no leader (its
        // error reaches at most k <= HALO cars back by the launch's end)
        if (lane == 31) xn = frel ? x[CPT - 1] + CPT + vmax + 1u : x[CPT - 1];  // (relative form: a free road ahead)
      } else {
        const uint32_t slot = phase++ & 1u;
        if (lane == 0) s_lead[slot][warp] = x[0];
        __syncthreads();
        xn = __shfl_down_sync(0xffffffffu, x[0], 1);
        if (lane == 31) xn = (warp + 1 < NW) ? s_lead[slot][warp + 1] : x[CPT - 1];
      }
      if (plain && !(base < bound && bound <= base + CPT)) {
        const uint32_t Q = mulmod_x2(P2, base < bound ? E : E2);
#if NB_TB_FREL && NB_TB_MN3
        if (frel) {
          // the same car update with the headway and the move as exact FP32
          // adds of the (relative, < 2^24) positions' bit patterns
#pragma unroll
          for (int c = 0; c < CPT; ++c) {
            const uint32_t s = mulmod_x2(c_apow2.v[c], Q);
            const uint32_t xl = (c + 1 < CPT) ? x[c + 1 < CPT ? c + 1 : c] : xn - CPT;
            const float gap = fadd_denorm(__uint_as_float(xl), -__uint_as_float(x[c]));
            int dec;
            asm("mul.hi.s32 %0, %1, 1;" : "=r"(dec) : "r"(static_cast<int>(tp * ra.neg1 + s)));
            float m3;
            asm("min.f32 %0, %1, %2, %3;" : "=f"(m3)
                : "f"(fadd_denorm(__uint_as_float(v[c]), __uint_as_float(1u))),
                  "f"(__uint_as_float(vmax)), "f"(gap));
            v[c] = static_cast<uint32_t>(max(static_cast<int>(__float_as_uint(m3)) + dec, 0));
            x[c] = __float_as_uint(fadd_denorm(__uint_as_float(x[c]), __uint_as_float(v[c])));
          }
        } else
#endif
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          // Balanced between the FMA and ALU pipes (both issue a warp
          // instruction every 2 cycles per SMSP): draw via mulmod_x2 (IMAD.WIDE
          // + LEA.HI + VIADDMNMX), headway x*(-1) + leader as one IMAD (neg1
          // is a launch parameter, so ptxas cannot turn it into an ALU IADD3;
          // measured +10 % on C3), deceleration flag as the sign of s - tp
          // (ptxas fuses it with the add: LEA.HI.SX32; forcing it onto the
          // FMA pipe as IMAD.HI measured 8 % slower).
          const uint32_t s = mulmod_x2(c_apow2.v[c], Q);
#if NB_TB_MN3
          // gap = x_{c+1} - x_c - 1 from the offset form (the next lane's
          // car 0 is not offset: minus CPT); tp * (-1) + s keeps s - tp an
          // IMAD (FMA pipe).  min(v + 1, vmax, gap) is ONE three-input
          // FMNMX3 on the integers' bit patterns (non-negative integers
          // order like the floats they encode; the NaN patterns of a gap
          // above 0x7f800000, or of the halo front car's meaningless gap,
          // lose every min), with v + 1 as an exact denormal FADD on the FP32
          // pipe: one ALU instruction where min/min took two.
          const uint32_t xl = (c + 1 < CPT) ? x[c + 1] : xn - CPT;
          const uint32_t gap = x[c] * ra.neg1 + xl;
          int dec;
          asm("mul.hi.s32 %0, %1, 1;" : "=r"(dec) : "r"(static_cast<int>(tp * ra.neg1 + s)));
          float m3;
          asm("min.f32 %0, %1, %2, %3;" : "=f"(m3)
              : "f"(fadd_denorm(__uint_as_float(v[c]), __uint_as_float(1u))),
                "f"(__uint_as_float(vmax)), "f"(__uint_as_float(gap)));
          v[c] = static_cast<uint32_t>(max(static_cast<int>(__float_as_uint(m3)) + dec, 0));
#else
          const uint32_t xl = (c + 1 < CPT) ? x[c + 1] : xn;
          const uint32_t d = x[c] * ra.neg1 + xl;
          int dec;
          asm("mul.hi.s32 %0, %1, 1;" : "=r"(dec) : "r"(static_cast<int>(s - tp)));
          const int vc = static_cast<int>(min(min(v[c] + 1, vmax), d - 1));
          v[c] = static_cast<uint32_t>(max(vc + dec, 0));
#endif
          x[c] += v[c];
        }
        if (own_all) {
#if NB_TB_VSUM == 1
          s_acc[j][threadIdx.x] += static_cast<Acc>(vsum_fp32<CPT>(v));
#elif NB_TB_VSUM == 2
          s_acc[j][threadIdx.x] += static_cast<Acc>(vsum_imad<CPT>(v));
#else
          s_acc[j][threadIdx.x] += static_cast<Acc>(VSum<uint32_t, CPT>::sum(v));
#endif
        } else if (own) {  // a shard's last, partial tile
          Acc sum = 0;
#pragma unroll
          for (int c = 0; c < CPT; ++c) sum += ((own >> c) & 1ull) ? v[c] : 0u;
          s_acc[j][threadIdx.x] += sum;
        }
      } else {
        // near the origin / at the rank seam / in the tile wrapping past id
        // N-1: per car, base E or E2 by rank side, a^-N for wrapped ids
        const uint32_t QE = mulmod_x2(P2, E), QE2 = mulmod_x2(P2, E2);
        const uint32_t QEw = mulmod_d(QE, ra.an_inv), QE2w = mulmod_d(QE2, ra.an_inv);
        Acc sum = 0;
        uint32_t crs = 0;
        if (frel) {  // the rank seam inside a relative tile: absolute for this step
          xn += xb;
#pragma unroll
          for (int c = 0; c < CPT; ++c) x[c] += xb;
        }
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const bool wrapped = base + c >= N;
          const uint32_t id = wrapped ? base + c - N : base + c;
          const uint32_t q = id < bound ? (wrapped ? QEw : QE) : (wrapped ? QE2w : QE2);
          const uint32_t s = mulmod_x2(c_apow2.v[c], q);
          uint32_t cr = 0;
#if NB_TB_MN3
          const uint32_t xl = (c + 1 < CPT) ? x[c + 1] + (c + 1) : xn;
          uint32_t xnew;
          v[c] = car_any(x[c] + c, xl, v[c], s, L, vmax, tp, xnew, cr);
          x[c] = xnew - c;
#else
          const uint32_t xl = (c + 1 < CPT) ? x[c + 1] : xn;
          v[c] = car_any(x[c], xl, v[c], s, L, vmax, tp, x[c], cr);
#endif
          const bool mine = (own >> c) & 1ull;
          sum += mine ? v[c] : 0u;
          crs += mine ? cr : 0u;
        }
        s_acc[j][threadIdx.x] += sum;
        if (crs) atomicAdd(&ra.rec[(t + j) % kRecCap].c, crs);
        if (frel) {
#pragma unroll
          for (int c = 0; c < CPT; ++c) x[c] -= xb;
        }
      }
    }
    if (frel) {
#pragma unroll
      for (int c = 0; c < CPT; ++c) x[c] += xb;
    }
#if NB_TB_MN3
#pragma unroll
    for (int c = 1; c < CPT; ++c) x[c] += c;
#endif
    if (fast) {
      // A shard's last tile may spill past nl into its halo/padding region,
      // which the plan kernel rewrites before the next launch reads it.
      if (u0 + CPT <= WSTORE) {
#pragma unroll
        for (int q = 0; q < CPT / 4; ++q)
          *reinterpret_cast<uint4*>(Xo + bl + 4 * q) =
              make_uint4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
        VLanes<VT, CPT>::store(Vo + bl, v);
      }
    } else {
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        if ((own >> c) & 1ull) {
          Xo[bl + c] = x[c];
          Vo[bl + c] = static_cast<VT>(v[c]);
        }
      }
    }
  }
  // Per-step velocity sums: warp w reduces steps w, w+NW, ...
  __syncthreads();
  for (uint32_t j = warp; j < k; j += NW) {
    unsigned long long acc = 0;
#pragma unroll
    for (int q = 0; q < TPB / 32; ++q) acc += s_acc[j][lane + 32 * q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0 && acc) atomicAdd(&ra.rec[(t + j) % kRecCap].sumv, acc);
  }
#ifdef NB_TB_TRACE
  if (threadIdx.x == 0) {
    const unsigned long long now = tb_now();
    atomicMin(trc + 2, now);
    atomicMax(trc + 3, now);
  }
#endif
  if (RANGE && !rg.epi) return;
  if (!last_block_done(ctl)) return;
#ifdef NB_TB_TRACE
  if (threadIdx.x == 0) trc[4] = tb_now();
#endif

  // Last block: check the plan, advance the control block, plan the next k.
  // One thread per step (k <= kPlanMax <= TPB), earliest mismatch wins.
  __shared__ uint32_t s_Wnext, s_bad;
  if (threadIdx.x == 0) s_bad = ~0u;
  __syncthreads();
  if (threadIdx.x < k) {
    const uint32_t j = threadIdx.x;
    StepRec* r = ra.rec + ((t + j) % kRecCap);
    const uint32_t c = __ldcg(&r->c);  // other blocks' atomics live in L2
    r->W = ctl->Wk[j];
    r->cplan = ctl->ck[j];
    // A shard sees only its own crossings; the host checks their sum.
    if (!ra.sharded && c != ctl->ck[j]) atomicMin(&s_bad, j);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_bad != ~0u && !ctl->err) {
      ctl->err = 1;
      ctl->err_step = static_cast<unsigned int>(t + s_bad);
    }
    uint32_t Wn = ctl->Wk[k - 1] + ctl->ck[k - 1];
    if (Wn >= N) Wn -= N;
    s_Wnext = Wn;
  }
  __syncthreads();
  const uint32_t Wn = s_Wnext;
  // The next plan: inline when its cone (kplan (vmax + 1) cars) fits this
  // block; otherwise the host enqueues a 256-thread cone kernel after this
  // launch (tb_plan_inline), and a segmented ring plans in its exchange
  // kernel (shard_kernels.cuh), which needs cars of other segments.
  const bool inline_plan = !ra.sharded && tb_plan_inline(ra.kplan, ra.vmax, TPB);
  if (inline_plan) {
    cone_plan<VT, TPB>(ra, Xo, Vo, t + k, Wn, ra.kplan, ctl);
    for (uint32_t j = threadIdx.x; j < ra.kplan; j += TPB) {
      StepRec* r = ra.rec + ((t + k + j) % kRecCap);
      r->sumv = 0;
      r->c = 0;
    }
  }
  if (threadIdx.x == 0) {
    ctl->W = Wn;
    ctl->t = t + k;
    ctl->buf = static_cast<unsigned int>(b ^ 1);
    ctl->ticket = 0;
  }
  if constexpr (PUSH) shard_push<VT, TPB>(ra, Xo, Vo, Wn, xa);
#ifdef NB_TB_TRACE
  __syncthreads();
  if (threadIdx.x == 0) trc[5] = tb_now();
#endif
}

template <typename VT, int TPB, int CPT, int HALO, bool WT>
__global__ void __launch_bounds__(TPB, NB_TB_MINB) nasch_tb_kernel(const RingArgs ra, const uint32_t k) {
  tb_body<VT, TPB, CPT, HALO, WT, false>(ra, k, XchgArgs{});
}

// Range launch of the streamed job (TbRange).
template <typename VT, int TPB, int CPT, int HALO, bool WT>
__global__ void __launch_bounds__(TPB, NB_TB_MINB)
    nasch_tb_range_kernel(const RingArgs ra, const uint32_t k, const TbRange rg) {
  tb_body<VT, TPB, CPT, HALO, WT, false, true>(ra, k, XchgArgs{}, rg);
}

// Segmented ring with the peer-memory exchange (sharded.cu, kXchgP2P).
template <typename VT, int TPB, int CPT, int HALO, bool WT>
__global__ void __launch_bounds__(TPB, NB_TB_MINB)
    nasch_tb_push_kernel(const RingArgs ra, const uint32_t k, const XchgArgs xa) {
  tb_body<VT, TPB, CPT, HALO, WT, true>(ra, k, xa);
}

}  // namespace nb200
