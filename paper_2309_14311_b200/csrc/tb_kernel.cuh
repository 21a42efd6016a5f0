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

// The launch body.  PUSH (segmented ring, peer-memory exchange only): the
// launch's last block also publishes this segment's exchange record for the
// next launch straight into every segment's receive slots (shard_push,
// shard_kernels.cuh) -- the pack and the all-gather fused into the step
// kernel.  PUSH = false compiles to the plain kernel (dead code removed).
template <typename VT, int TPB, int CPT, int HALO, bool WT, bool PUSH>
__device__ __forceinline__ void tb_body(const RingArgs& ra, const uint32_t k, const XchgArgs& xa) {
  using G = TbGeom<TPB, CPT, HALO, WT>;
  constexpr uint32_t LOAD = G::kLoad;     // cars spanned per block tile
  constexpr uint32_t STORE = G::kStore;   // cars owned (stored) per block tile
  constexpr uint32_t WSTORE = G::kWarpStore;  // owned per halo unit (warp or block)
  constexpr int NW = TPB / 32;
  static_assert(HALO >= kPlanMax && HALO % 16 == 0, "halo must cover the plan");
  using Acc = typename std::conditional<sizeof(VT) == 1, uint32_t, unsigned long long>::type;
  __shared__ uint32_t s_W[kPlanMax], s_E[kPlanMax], s_E2[kPlanMax];
  __shared__ uint32_t s_lead[2][NW];
  __shared__ Acc s_acc[kPlanMax][TPB];  // per-thread, per-step velocity sums

  Ctl* ctl = ra.ctl;
  const uint32_t N = ra.n, L = ra.L, vmax = ra.vmax, tp = ra.tp;
  const uint64_t t = ctl->t;
  const int b = static_cast<int>(ctl->buf);
  if (threadIdx.x < kPlanMax) {
    s_W[threadIdx.x] = ctl->Wk[threadIdx.x];
    s_E[threadIdx.x] = ctl->Ek[threadIdx.x];
    s_E2[threadIdx.x] = ctl->E2k[threadIdx.x];
  }
#pragma unroll
  for (int j = 0; j < kPlanMax; ++j) s_acc[j][threadIdx.x] = 0;
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

  // P = a^(global id of this thread's first car in its first tile)
  uint32_t P = mulmod_d(mulmod_d(ra.agofs, __ldg(ra.blkpow + blockIdx.x)), __ldg(ra.thrpow + threadIdx.x));
  uint32_t phase = 0;  // running step counter across tiles: s_lead slot parity
  const uint32_t nl = ra.nl;  // cars stored here (a shard's segment, or the ring)
  const uint32_t ntiles = (nl + STORE - 1) / STORE;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t a0 = tile * STORE;          // local index of the tile
    const uint32_t bl = a0 + i0;               // local index of car 0
    const uint32_t base = ra.gofs + bl;        // global id of car 0 (may exceed N at the wrap)
    const bool nowrap = ra.gofs + a0 + LOAD <= N;  // block-uniform: ids do not wrap
    // Contiguous in memory: always for a shard (its halo sits inline after
    // nl); on one GPU unless the tile wraps past id N-1.
    const bool fast = ra.sharded || nowrap;
    uint32_t x[CPT], v[CPT], ap[CPT];
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
    // 2 * a^id for this thread's cars (doubled for mulmod_x2): a^(first
    // id) times a^c from the constant table -- independent products, no
    // dependent chain.  Ids wrapped past N (only in the tile straddling id
    // N-1) also multiply by a^-N.
    ap[0] = P << 1;
#pragma unroll
    for (int c = 1; c < CPT; ++c) ap[c] = mulmod_d(P, c_pow.lin[c]) << 1;
    if (!nowrap) {
#pragma unroll
      for (int c = 0; c < CPT; ++c)
        if (base + c >= N) ap[c] = mulmod_d(ap[c] >> 1, ra.an_inv) << 1;
    }
    P = mulmod_d(P, ra.g);
    // bit c: car c is stored by this tile (all of them but in the halo and
    // at a shard's end)
    const bool own_all = u0 + CPT <= WSTORE && bl + CPT <= nl;
    uint32_t own = own_all ? (1u << CPT) - 1u : 0u;
    if (!own_all) {
#pragma unroll
      for (int c = 0; c < CPT; ++c) own |= (u0 + c < WSTORE && bl + c < nl) ? (1u << c) : 0u;
    }
    uint32_t xmax = x[0];
#pragma unroll
    for (int c = 1; c < CPT; ++c) xmax = max(xmax, x[c]);
    const bool plain = nowrap && xmax < L - reach;

    for (uint32_t j = 0; j < k; ++j) {
      const uint32_t E = s_E[j], E2 = s_E2[j];
      const uint32_t bound = N - s_W[j];  // id of the rank-0 car (N when W = 0)
      // Slots alternate with the running step count, so one barrier per step
      // suffices (a slot is rewritten only after the next barrier).
      uint32_t xn;
      if (WT) {
        xn = __shfl_down_sync(0xffffffffu, x[0], 1);
        // warp tiles: the front car of the warp's halo has no leader (its
        // error reaches at most k <= HALO cars back by the launch's end)
        if (lane == 31) xn = x[CPT - 1];
      } else {
        const uint32_t slot = phase++ & 1u;
        if (lane == 0) s_lead[slot][warp] = x[0];
        __syncthreads();
        xn = __shfl_down_sync(0xffffffffu, x[0], 1);
        if (lane == 31) xn = (warp + 1 < NW) ? s_lead[slot][warp + 1] : x[CPT - 1];
      }
      if (plain && !(base < bound && bound <= base + CPT)) {
        const uint32_t Es = base < bound ? E : E2;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          // Balanced between the FMA and ALU pipes (both issue a warp
          // instruction every 2 cycles per SMSP): draw via mulmod_x2 (IMAD.WIDE
          // + LEA.HI + VIADDMNMX), headway x*(-1) + leader as one IMAD (neg1
          // is a launch parameter, so ptxas cannot turn it into an ALU IADD3;
          // measured +10 % on C3), deceleration flag as the sign of s - tp
          // (ptxas fuses it with the add: LEA.HI.SX32; forcing it onto the
          // FMA pipe as IMAD.HI measured 8 % slower).
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
        } else if (own) {  // a shard's last, partial tile
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
          uint32_t id = base + c;
          if (id >= N) id -= N;
          const uint32_t s = mulmod_x2(ap[c], id < bound ? E : E2);
          const uint32_t xl = (c + 1 < CPT) ? x[c + 1] : xn;
          uint32_t cr = 0;
          v[c] = car_any(x[c], xl, v[c], s, L, vmax, tp, x[c], cr);
          const bool mine = (own >> c) & 1u;
          sum += mine ? v[c] : 0u;
          crs += mine ? cr : 0u;
        }
        s_acc[j][threadIdx.x] += sum;
        if (crs) atomicAdd(&ra.rec[(t + j) % kRecCap].c, crs);
      }
    }
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
        if ((own >> c) & 1u) {
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
  if (!last_block_done(ctl)) return;

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
  if (ra.sharded) {
    // The next plan needs cars of other shards: the exchange + plan kernel
    // (shard_kernels.cuh) produce it.
    if (threadIdx.x == 0) {
      ctl->W = Wn;
      ctl->t = t + k;
      ctl->buf = static_cast<unsigned int>(b ^ 1);
      ctl->ticket = 0;
    }
    if constexpr (PUSH) shard_push<VT, TPB>(ra, Xo, Vo, Wn, xa);
    return;
  }
  cone_plan<VT, TPB>(ra, Xo, Vo, t + k, Wn, ra.kplan, ctl);
  for (uint32_t j = threadIdx.x; j < ra.kplan; j += TPB) {
    StepRec* r = ra.rec + ((t + k + j) % kRecCap);
    r->sumv = 0;
    r->c = 0;
  }
  if (threadIdx.x == 0) {
    ctl->W = Wn;
    ctl->t = t + k;
    ctl->buf = static_cast<unsigned int>(b ^ 1);
    ctl->ticket = 0;
  }
}

template <typename VT, int TPB, int CPT, int HALO, bool WT>
__global__ void __launch_bounds__(TPB, NB_TB_MINB) nasch_tb_kernel(const RingArgs ra, const uint32_t k) {
  tb_body<VT, TPB, CPT, HALO, WT, false>(ra, k, XchgArgs{});
}

// Segmented ring with the peer-memory exchange (sharded.cu, kXchgP2P).
template <typename VT, int TPB, int CPT, int HALO, bool WT>
__global__ void __launch_bounds__(TPB, NB_TB_MINB)
    nasch_tb_push_kernel(const RingArgs ra, const uint32_t k, const XchgArgs xa) {
  tb_body<VT, TPB, CPT, HALO, WT, true>(ra, k, xa);
}

}  // namespace nb200
