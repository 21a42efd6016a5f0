// ensemble_tb.cuh -- the ensemble (BASELINE config 4: thousands of
// independent rings) run through the temporal-blocked warp-tile step of the
// single-ring kernel (tb_kernel.cuh) instead of one shared-memory CTA per
// ring: every ring is cut into warp tiles of 496 owned cars + a 16-car halo,
// all tiles of all rings are advanced K <= 16 steps per launch from
// registers, and a planner launch before each step launch computes every
// ring's origin-cone plan in one warp per ring (cone_warp.cuh), checks the
// previous launch's crossing counts against it and folds the per-step
// velocity sums.
//
// Per ring r: EnsRing (parameters, step counter, rank offset, parity), a
// Ctl used as its plan (W, E, E2, c for each planned step) and EnsCount
// (per-step crossings and velocity sums accumulated by the tiles).  Rings
// step in lock-step launches but each plans min(K, its remaining steps), so
// rings with fewer configured steps simply stop.
#pragma once
#include <cstdint>

#include "cone_warp.cuh"
#include "step_kernels.cuh"

namespace nb200 {

// Plain-path car update (tb_kernel.cuh): velocity sums as FP32 denormal
// adds, min(v + 1, vmax, gap) as one FMNMX3 on offset positions.
#ifndef NB_ET_VSUM
#define NB_ET_VSUM 1
#endif
#ifndef NB_ET_MN3
#define NB_ET_MN3 1
#endif
constexpr int kEtTPB = 128;
#ifndef NB_ET_HALO
#define NB_ET_HALO 32
#endif
constexpr int kEtCPT = 16;
constexpr uint32_t kEtHalo = NB_ET_HALO;              // = the deepest launch
constexpr uint32_t kEtLoad = 32u * kEtCPT;            // cars spanned by a warp tile
constexpr uint32_t kEtStore = kEtLoad - kEtHalo;      // owned (496 with a 16-car halo)
constexpr uint32_t kEtK = kEtHalo;                    // steps per launch (<= halo)

struct EnsRing {
  unsigned long long off;         // first car in X / V (multiple of 16)
  unsigned long long t;           // steps done
  unsigned long long steps;       // configured total
  unsigned long long sumv_total;  // sum over completed steps of sum(v)
  uint32_t n, L, vmax, tp, s0, an, an_inv;
  uint32_t W;          // rank offset at t
  uint32_t buf;        // which of X[2] / V[2] holds the state at t
  uint32_t k;          // steps planned for the pending launch (0: none)
  uint32_t last_sumv;  // velocity sum after the last completed step
  uint32_t err;        // counted crossings contradicted the plan
};

struct EnsCount {
  unsigned long long sumv[kEtK];
  uint32_t c[kEtK];
};

struct EnsTile {
  uint32_t ring;
  uint32_t base;   // local id of the tile's first car
  uint32_t abase;  // a^base mod m
  uint32_t pad;
};

struct EnsArgs {
  EnsRing* rings;
  Ctl* plans;
  EnsCount* counts;
  const EnsTile* tiles;
  uint32_t nrings, ntiles;
  uint32_t* X[2];
  uint8_t* V[2];
  const uint32_t* thrpow;  // a^(lane * kEtCPT)
  uint32_t neg1;           // -1 as a launch parameter (see tb_kernel.cuh)
};

// One warp per ring: fold the finished launch (verify crossings, add the
// velocity sums, advance t / W / parity), then plan min(kreq, remaining)
// steps from the current state.  kreq = 0 only folds.
__global__ void __launch_bounds__(256) ens_plan_kernel(const EnsArgs ea, const uint32_t kreq) {
  __shared__ ConeTab tab;
  cone_tab_fill_lin(tab);
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= ea.nrings) return;
  EnsRing& rd = ea.rings[r];
  Ctl* pl = ea.plans + r;
  EnsCount* cn = ea.counts + r;
  const uint32_t N = rd.n;
  const uint32_t kp = rd.k;
  if (kp) {
    uint32_t bad = 0;
    unsigned long long sv = 0;
    if (lane < kp) {
      bad = cn->c[lane] != pl->ck[lane];
      sv = cn->sumv[lane];
    }
    const unsigned long long last = __shfl_sync(0xffffffffu, sv, kp - 1);
    for (int o = 16; o > 0; o >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
    bad = __reduce_or_sync(0xffffffffu, bad);
    uint32_t Wn = pl->Wk[kp - 1] + pl->ck[kp - 1];
    if (Wn >= N) Wn -= N;
    __syncwarp();
    if (lane == 0) {
      if (bad) rd.err = 1;
      rd.sumv_total += sv;
      rd.last_sumv = static_cast<uint32_t>(last);
      rd.W = Wn;
      rd.t += kp;
      rd.buf ^= 1u;
      rd.k = 0;
    }
    if (lane < kEtK) {
      cn->c[lane] = 0;
      cn->sumv[lane] = 0;
    }
    __syncwarp();
  }
  const unsigned long long remain = rd.steps - rd.t;
  const uint32_t k = static_cast<uint32_t>(remain < kreq ? remain : kreq);
  if (k == 0) return;
  RingArgs ra{};
  ra.n = N;
  ra.L = rd.L;
  ra.vmax = rd.vmax;
  ra.tp = rd.tp;
  ra.s0 = rd.s0;
  ra.an = rd.an;
  ra.an_inv = rd.an_inv;
  const bool b = rd.buf != 0;  // ternaries: a runtime index into the by-value args would go to the stack
  cone_warp<uint8_t, false>(ra, (b ? ea.X[1] : ea.X[0]) + rd.off, (b ? ea.V[1] : ea.V[0]) + rd.off, rd.t, rd.W,
                            k, 0, k, pl, tab);
  __syncwarp();
  if (lane == 0) rd.k = k;
}

template <int TPB>
#ifndef NB_ET_MINB
#define NB_ET_MINB 4
#endif
__global__ void __launch_bounds__(TPB, NB_ET_MINB) ens_tb_kernel(const EnsArgs ea) {
  constexpr int CPT = kEtCPT;
  constexpr int NW = TPB / 32;
  __shared__ uint32_t s_acc[kEtK][TPB];  // per-thread per-step velocity sums (u8 lanes)
  __shared__ uint32_t s_plan[NW][3][kEtK];  // the warp's ring plan: W, E, E2 per step
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < int(kEtK); ++j) s_acc[j][threadIdx.x] = 0;
  const uint32_t ap_lane = __ldg(ea.thrpow + lane);
  for (uint32_t wt = blockIdx.x * NW + warp; wt < ea.ntiles; wt += gridDim.x * NW) {
    const EnsTile td = ea.tiles[wt];
    const EnsRing* rp = ea.rings + td.ring;
    const uint32_t k = rp->k;
    if (k == 0) continue;  // warp-uniform
    const uint32_t N = rp->n, L = rp->L, vmax = rp->vmax, tp = rp->tp, an_inv = rp->an_inv;
    const unsigned long long off = rp->off;
    const bool b = rp->buf != 0;
    const Ctl* pl = ea.plans + td.ring;
    if (lane < k) {
      s_plan[warp][0][lane] = pl->Wk[lane];
      s_plan[warp][1][lane] = pl->Ek[lane];
      s_plan[warp][2][lane] = pl->E2k[lane];
    }
    __syncwarp();
    const uint32_t* X = (b ? ea.X[1] : ea.X[0]) + off;
    const uint8_t* V = (b ? ea.V[1] : ea.V[0]) + off;

    const uint32_t u0 = lane * CPT;
    const uint32_t base = td.base + u0;  // local id of car 0 (may pass N in the ring's last tile)
    const bool nowrap = td.base + kEtLoad <= N;  // warp-uniform
    uint32_t x[CPT], v[CPT], ap[CPT];
    if (nowrap) {
#pragma unroll
      for (int q = 0; q < CPT / 4; ++q) {
        const uint4 r4 = ld_nc_v4(X + base + 4 * q);
        x[4 * q] = r4.x;
        x[4 * q + 1] = r4.y;
        x[4 * q + 2] = r4.z;
        x[4 * q + 3] = r4.w;
      }
      VLanes<uint8_t, CPT>::load(V + base, v);
    } else {
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        uint32_t id = base + c;
        while (id >= N) id -= N;  // a ring shorter than its tile wraps more than once
        x[c] = X[id];
        v[c] = V[id];
      }
    }
    const uint32_t P = mulmod_d(td.abase, ap_lane);  // a^base
    ap[0] = P << 1;
#pragma unroll
    for (int c = 1; c < CPT; ++c) ap[c] = mulmod_d(P, c_pow.lin[c]) << 1;
    if (!nowrap) {
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        uint32_t id = base + c, a = ap[c] >> 1;
        while (id >= N) {
          id -= N;
          a = mulmod_d(a, an_inv);
        }
        ap[c] = a << 1;
      }
    }
    const bool own_all = u0 + CPT <= kEtStore && base + CPT <= N;
    uint32_t own = own_all ? (1u << CPT) - 1u : 0u;
    if (!own_all) {
#pragma unroll
      for (int c = 0; c < CPT; ++c) own |= (u0 + c < kEtStore && base + c < N) ? (1u << c) : 0u;
    }
    uint32_t xmax = x[0];
#pragma unroll
    for (int c = 1; c < CPT; ++c) xmax = max(xmax, x[c]);
    // this thread's ids run consecutively below N (only the ring's last
    // tile has threads that wrap)
    const bool plain = base + CPT <= N && xmax < L - k * vmax;
#if NB_ET_MN3
    // offset form x[c] - c for the plain path's FMNMX3 (tb_kernel.cuh)
#pragma unroll
    for (int c = 1; c < CPT; ++c) x[c] -= c;
#endif
    for (uint32_t j = 0; j < k; ++j) {
      const uint32_t E = s_plan[warp][1][j], E2 = s_plan[warp][2][j];
      const uint32_t bound = N - s_plan[warp][0][j];
      uint32_t xn = __shfl_down_sync(0xffffffffu, x[0], 1);
      if (lane == 31) xn = x[CPT - 1];  // tile front: unknown leader, k <= halo
      const bool tplain = plain && !(base < bound && bound <= base + CPT);
      if (__all_sync(0xffffffffu, tplain)) {
        const uint32_t Es = base < bound ? E : E2;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const uint32_t s = mulmod_x2(ap[c], Es);
#if NB_ET_MN3
          const uint32_t xl = (c + 1 < CPT) ? x[c + 1] : xn - CPT;
          const uint32_t gap = x[c] * ea.neg1 + xl;
          int dec;
          asm("mul.hi.s32 %0, %1, 1;" : "=r"(dec) : "r"(static_cast<int>(tp * ea.neg1 + s)));
          float m3;
          asm("min.f32 %0, %1, %2, %3;" : "=f"(m3)
              : "f"(fadd_denorm(__uint_as_float(v[c]), __uint_as_float(1u))),
                "f"(__uint_as_float(vmax)), "f"(__uint_as_float(gap)));
          v[c] = static_cast<uint32_t>(max(static_cast<int>(__float_as_uint(m3)) + dec, 0));
#else
          const uint32_t xl = (c + 1 < CPT) ? x[c + 1] : xn;
          const uint32_t d = x[c] * ea.neg1 + xl;
          const int vc = static_cast<int>(min(min(v[c] + 1, vmax), d - 1));
          int dec;
          asm("mul.hi.s32 %0, %1, 1;" : "=r"(dec) : "r"(static_cast<int>(s - tp)));
          v[c] = static_cast<uint32_t>(max(vc + dec, 0));
#endif
          x[c] += v[c];
        }
        if (own_all) {  // separate branches (as tb_kernel.cuh): no per-car selects
#if NB_ET_VSUM
          s_acc[j][threadIdx.x] += vsum_fp32<CPT>(v);
#else
          s_acc[j][threadIdx.x] += VSum<uint32_t, CPT>::sum(v);
#endif
        } else if (own) {
          uint32_t sum = 0;
#pragma unroll
          for (int c = 0; c < CPT; ++c) sum += ((own >> c) & 1u) ? v[c] : 0u;
          s_acc[j][threadIdx.x] += sum;
        }
      } else {
        uint32_t sum = 0, crs = 0;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          uint32_t id = base + c;
          while (id >= N) id -= N;
          const uint32_t s = mulmod_x2(ap[c], id < bound ? E : E2);
#if NB_ET_MN3
          const uint32_t xc = x[c] + c;
          const uint32_t xl = (c + 1 < CPT) ? x[c + 1] + (c + 1) : xn;
#else
          const uint32_t xc = x[c];
          const uint32_t xl = (c + 1 < CPT) ? x[c + 1] : xn;
#endif
          uint32_t d = xc * ea.neg1 + xl;
          d = min(d, d + L);  // leader past the origin: + L
          const int vc = static_cast<int>(min(min(v[c] + 1, vmax), d - 1));
          int dec;
          asm("mul.hi.s32 %0, %1, 1;" : "=r"(dec) : "r"(static_cast<int>(s - tp)));
          v[c] = static_cast<uint32_t>(max(vc + dec, 0));
          const uint32_t xs = xc + v[c];
#if NB_ET_MN3
          x[c] = min(xs, xs - L) - c;
#else
          x[c] = min(xs, xs - L);
#endif
          const bool mine = (own >> c) & 1u;
          sum += mine ? v[c] : 0u;
          crs += (mine && xs >= L) ? 1u : 0u;
        }
        s_acc[j][threadIdx.x] += sum;
        crs = __reduce_add_sync(0xffffffffu, crs);
        if (lane == 0 && crs) atomicAdd(&ea.counts[td.ring].c[j], crs);
      }
    }
#if NB_ET_MN3
#pragma unroll
    for (int c = 1; c < CPT; ++c) x[c] += c;
#endif
    // Per-step sums of this tile: one atomic per step.
    for (uint32_t j = 0; j < k; ++j) {
      const uint32_t sv = __reduce_add_sync(0xffffffffu, s_acc[j][threadIdx.x]);
      s_acc[j][threadIdx.x] = 0;
      if (lane == 0 && sv) atomicAdd(&ea.counts[td.ring].sumv[j], static_cast<unsigned long long>(sv));
    }
    // output pointers rebuilt here (kernel parameters + the ring's offset)
    // rather than kept live through the step loop
    const unsigned long long off2 = rp->off;
    const bool b2 = rp->buf != 0;
    uint32_t* Xo = (b2 ? ea.X[0] : ea.X[1]) + off2;
    uint8_t* Vo = (b2 ? ea.V[0] : ea.V[1]) + off2;
    if (own_all && nowrap) {
#pragma unroll
      for (int q = 0; q < CPT / 4; ++q)
        *reinterpret_cast<uint4*>(Xo + base + 4 * q) = make_uint4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
      VLanes<uint8_t, CPT>::store(Vo + base, v);
    } else {
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        if ((own >> c) & 1u) {
          Xo[base + c] = x[c];
          Vo[base + c] = static_cast<uint8_t>(v[c]);
        }
      }
    }
  }
}

}  // namespace nb200
