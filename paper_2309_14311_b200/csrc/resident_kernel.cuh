// resident_kernel.cuh -- small rings (N <= 4096): the whole ring lives in
// one CTA's shared memory for all the steps of a launch.
//
// Below the temporal-blocking threshold a per-step launch costs far more
// than the step itself (BASELINE config 1: 200 cars).  One 1024-thread
// block loads the ring once, runs `steps` steps with two barriers each --
// exactly the rank/draw bookkeeping of step_kernels.cuh, folded per step by
// every warp from per-warp crossing counts -- records every step's exact
// velocity sum, crossing count and rank offset, and writes the ring back
// in place.
#pragma once
#include <cstdint>

#include "step_kernels.cuh"

namespace nb200 {

constexpr uint32_t kResidentMaxCars = 4096;

template <typename VT, int TPB>
__global__ void __launch_bounds__(TPB, 1) ring_resident_kernel(const RingArgs ra, const uint32_t steps) {
  __shared__ uint32_t sx[kResidentMaxCars];
  __shared__ uint32_t sv[kResidentMaxCars];
  __shared__ uint32_t apw[256];
  __shared__ uint32_t slot_c[2][TPB / 32], slot_v[2][TPB / 32];
  __shared__ uint32_t s_lead[2][TPB];
  Ctl* ctl = ra.ctl;
  const uint32_t N = ra.n, L = ra.L, vmax = ra.vmax, tp = ra.tp;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint64_t t0 = ctl->t;
  const int b = static_cast<int>(ctl->buf);
  uint32_t* X = xbuf(ra, b);
  VT* V = vbuf_w<VT>(ra, b);
  for (uint32_t i = tid; i < 256; i += TPB) apw[i] = c_pow.lin[i];
  for (uint32_t i = tid; i < N; i += TPB) {
    sx[i] = X[i];
    sv[i] = static_cast<uint32_t>(V[i]);
  }
  uint32_t cpt = (N + TPB - 1) / TPB;
  cpt |= 1u;  // odd stride: conflict-free banks
  const uint32_t first = tid * cpt;
  const uint32_t cnt = first < N ? min(cpt, N - first) : 0u;
  const uint32_t next_tid = (first + cnt >= N) ? 0u : tid + 1;  // owner of the run's leader
  const uint32_t ap0 = cnt ? powmod(kA, first) : 1u;
  uint32_t W = ctl->W, E = ctl->E;
  __syncthreads();
  // One barrier per step (see ensemble.cu): runs publish their first
  // position in a parity-alternating slot read by the thread behind.
  for (uint32_t st = 0; st <= steps; ++st) {
    const uint32_t par = st & 1u;
    if (st < steps && cnt) s_lead[par][tid] = sx[first];
    __syncthreads();
    if (st > 0) {
      const uint32_t p = par ^ 1u;
      const uint32_t c = __reduce_add_sync(0xffffffffu, lane < TPB / 32 ? slot_c[p][lane] : 0u);
      const uint32_t sum = __reduce_add_sync(0xffffffffu, lane < TPB / 32 ? slot_v[p][lane] : 0u);
      uint32_t Wn = W + c;
      const bool wrap = Wn >= N;
      if (wrap) Wn -= N;
      if (tid == 0) {
        StepRec* r = ra.rec + ((t0 + st - 1) % kRecCap);
        r->sumv = sum;
        r->c = c;
        r->W = W;
      }
      const uint32_t ac = c < 256 ? apw[c] : powmod(kA, c);
      E = mulmod_d(E, wrap ? ac : mulmod_d(ra.an, ac));
      W = Wn;
      if (ra.dump) {  // checksum batch: step st-1's row in rank order
        uint32_t* row = ra.dump + size_t(st - 1) * 2u * N;
        for (uint32_t id = first; id < first + cnt; ++id) {
          uint32_t r = id + W;
          if (r >= N) r -= N;
          row[r] = sx[id];
          row[N + r] = sv[id];
        }
      }
    }
    if (st == steps) break;
    const uint32_t E2 = mulmod_d(E, ra.an_inv);
    const uint32_t bound = N - W;
    const uint32_t lead = cnt ? s_lead[par][next_tid] : 0u;
    uint32_t crs = 0, sum = 0;
    // plain run: no rank seam at or inside it, farthest car short of L
    const bool plain = cnt && !(first < bound && bound <= first + cnt) &&
                       sx[first + cnt - 1] + vmax < L;
    if (plain) {
      uint32_t s = mulmod_d(ap0, first < bound ? E : E2);
      uint32_t cx = sx[first];
      for (uint32_t c = 0; c < cnt; ++c) {
        const uint32_t id = first + c;
        if (c) s = mulmod_d(s, kA);
        const uint32_t nx = (c + 1 < cnt) ? sx[id + 1] : lead;
        uint32_t vn = min(min(sv[id] + 1, vmax), nx - cx - 1);
        if (s < tp) vn = static_cast<uint32_t>(max(static_cast<int>(vn) - 1, 0));
        sx[id] = cx + vn;
        sv[id] = vn;
        sum += vn;
        cx = nx;
      }
    } else if (cnt) {
      uint32_t s = mulmod_d(ap0, first < bound ? E : E2);
      uint32_t cx = sx[first];
      for (uint32_t c = 0; c < cnt; ++c) {
        const uint32_t id = first + c;
        if (c) s = mulmod_d(s, id == bound ? ra.a1 : kA);
        const uint32_t nx = (c + 1 < cnt) ? sx[id + 1] : lead;
        uint32_t xn;
        const uint32_t vn = car_any(cx, nx, sv[id], s, L, vmax, tp, xn, crs);
        sx[id] = xn;
        sv[id] = vn;
        sum += vn;
        cx = nx;
      }
    }
    crs = __reduce_add_sync(0xffffffffu, crs);
    sum = __reduce_add_sync(0xffffffffu, sum);
    if (lane == 0) {
      slot_c[par][warp] = crs;
      slot_v[par][warp] = sum;
    }
  }
  for (uint32_t i = tid; i < N; i += TPB) {
    X[i] = sx[i];
    V[i] = static_cast<VT>(sv[i]);
  }
  if (tid == 0) {
    StepRec* nrec = ra.rec + ((t0 + steps) % kRecCap);
    nrec->sumv = 0;
    nrec->c = 0;
    ctl->t = t0 + steps;
    ctl->W = W;
    ctl->E = E;
    ctl->E2 = mulmod_d(E, ra.an_inv);
  }
}

// Tiny rings (N <= 32 * CPW): one warp keeps every car in registers (CPW
// consecutive cars per lane) for a whole chunk of steps -- no barrier at
// all: leaders by shuffle (the leader of car N-1 is lane 0's first car),
// crossing count and velocity sum by warp reductions, W and E advanced by
// every lane.  Each car's draw multiplier is its own register (a^id, and
// a^(id-N) for the far side of the rank seam), so the draws of a lane's
// cars are independent products rather than a chain.  BASELINE config 1
// (200 cars) is bound by this per-step latency.
//
// EXACT (N a multiple of CPW, e.g. C1: 200 = 25 x 8): every lane holds CPW
// live cars or none, so the per-car work has no liveness predicate and no
// leader select -- the last live lane's external leader is car 0, chosen
// once per step -- and the dead lanes' sums are masked once per step.
template <typename VT, int CPW, bool EXACT = false>
__global__ void __launch_bounds__(32, 1) ring_warp_kernel(const RingArgs ra, const uint32_t steps) {
  __shared__ uint32_t apw[256];
  Ctl* ctl = ra.ctl;
  const uint32_t N = ra.n, L = ra.L, vmax = ra.vmax, tp = ra.tp;
  const uint32_t lane = threadIdx.x;
  const uint64_t t0 = ctl->t;
  const int b = static_cast<int>(ctl->buf);
  uint32_t* X = xbuf(ra, b);
  VT* V = vbuf_w<VT>(ra, b);
  for (uint32_t i = lane; i < 256; i += 32) apw[i] = c_pow.lin[i];
  uint32_t x[CPW], v[CPW], apA[CPW], apB[CPW];
  uint32_t live = 0;  // bit c: car lane*CPW + c exists
  const uint32_t first = lane * CPW;
  const uint32_t a0 = first < N ? powmod(kA, first) : 1u;
#pragma unroll
  for (int c = 0; c < CPW; ++c) {
    const uint32_t id = first + c;
    const bool ok = id < N;
    live |= ok ? (1u << c) : 0u;
    x[c] = ok ? X[id] : 0u;
    v[c] = ok ? static_cast<uint32_t>(V[id]) : 0u;
    const uint32_t a = mulmod(a0, c_pow.lin[c]);
    apA[c] = a << 1;
    apB[c] = mulmod(a, ra.an_inv) << 1;
  }
  // the lane holding car N-1 and its slot
  const uint32_t last_lane = (N - 1) / CPW, last_c = (N - 1) % CPW;
  // Next draw base for c = lane crossings, both cases, doubled for
  // mulmod_x2: E' = E a^c when W wraps past N, else E a^(N+c).  Each step
  // computes both candidates while its cars move, so the serial chain after
  // the crossing count is one shuffle (c < 32; larger counts take the table).
  const uint32_t candw2 = c_pow.lin[lane] << 1;
  const uint32_t candn2 = mulmod(ra.an, c_pow.lin[lane]) << 1;
  uint32_t W = ctl->W, E = ctl->E;
  uint32_t rsum = 0, rc = 0, rW = 0;  // batched step record (lane = step mod 32)
  __syncwarp();
  for (uint32_t st = 0; st < steps; ++st) {
    const uint32_t bound = N - W;
    const uint32_t nextw = mulmod_x2(candw2, E), nextn = mulmod_x2(candn2, E);
    uint32_t xn = __shfl_down_sync(0xffffffffu, x[0], 1);
    const uint32_t x00 = __shfl_sync(0xffffffffu, x[0], 0);  // leader of car N-1
    uint32_t sum = 0, crs = 0;
    if constexpr (EXACT) {
      if (lane == last_lane) xn = x00;
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        const uint32_t s = mulmod_x2(first + c < bound ? apA[c] : apB[c], E);
        const uint32_t xl = c + 1 < CPW ? x[c + 1] : xn;
        uint32_t d = xl - x[c];
        d = min(d, d + L);  // leader past the origin: + L
        const int vc = static_cast<int>(min(min(v[c] + 1, vmax), d - 1));
        int dec;
        asm("mul.hi.s32 %0, %1, 1;" : "=r"(dec) : "r"(static_cast<int>(s - tp)));
        v[c] = static_cast<uint32_t>(max(vc + dec, 0));
        const uint32_t xs = x[c] + v[c];
        x[c] = min(xs, xs - L);
        sum += v[c];
        crs += xs >= L ? 1u : 0u;
      }
      if (!live) sum = crs = 0;  // dead lane
    } else
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
      const uint32_t id = first + c;
      const uint32_t s = mulmod_x2(id < bound ? apA[c] : apB[c], E);
      const uint32_t xl = (lane == last_lane && c == int(last_c)) ? x00 : (c + 1 < CPW ? x[c + 1] : xn);
      uint32_t d = xl - x[c];
      d = min(d, d + L);  // leader past the origin (or N = 1: d = 0, gap = L - 1 via vmax <= L - 1)
      const int vc = static_cast<int>(min(min(v[c] + 1, vmax), d - 1));
      const int vnew = max(vc - (s < tp ? 1 : 0), 0);
      const uint32_t xs = x[c] + static_cast<uint32_t>(vnew);
      const bool ok = (live >> c) & 1u;
      if (ok) {
        v[c] = static_cast<uint32_t>(vnew);
        x[c] = min(xs, xs - L);
        sum += v[c];
        crs += xs >= L ? 1u : 0u;
      }
    }
    const uint32_t cj = __reduce_add_sync(0xffffffffu, crs);
    sum = __reduce_add_sync(0xffffffffu, sum);
    // Step records in batches of 32: lane (st mod 32) keeps this step's,
    // and the warp stores 32 at once (no per-step store on the chain).
    if (lane == (st & 31u)) {
      rsum = sum;
      rc = cj;
      rW = W;
    }
    if ((st & 31u) == 31u || st + 1 == steps) {
      if (lane <= (st & 31u)) {
        StepRec* r = ra.rec + ((t0 + (st & ~31u) + lane) % kRecCap);
        r->sumv = rsum;
        r->c = rc;
        r->W = rW;
      }
    }
    uint32_t Wn = W + cj;
    const bool wrap = Wn >= N;
    if (wrap) Wn -= N;
    const uint32_t fast = __shfl_sync(0xffffffffu, wrap ? nextw : nextn, cj & 31u);
    if (cj < 32) {
      E = fast;
    } else {
      const uint32_t ac = cj < 256 ? apw[cj] : powmod(kA, cj);
      E = mulmod_d(E, wrap ? ac : mulmod_d(ra.an, ac));
    }
    W = Wn;
    if (ra.dump) {  // checksum batch: this step's row in rank order
      uint32_t* row = ra.dump + size_t(st) * 2u * N;
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        if ((live >> c) & 1u) {
          uint32_t r = first + c + W;
          if (r >= N) r -= N;
          row[r] = x[c];
          row[N + r] = v[c];
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < CPW; ++c) {
    if ((live >> c) & 1u) {
      X[first + c] = x[c];
      V[first + c] = static_cast<VT>(v[c]);
    }
  }
  if (lane == 0) {
    StepRec* nrec = ra.rec + ((t0 + steps) % kRecCap);
    nrec->sumv = 0;
    nrec->c = 0;
    ctl->t = t0 + steps;
    ctl->W = W;
    ctl->E = E;
    ctl->E2 = mulmod_d(E, ra.an_inv);
  }
}

// Small rings of up to 512 cars on FOUR warps, one per SM sub-partition
// (CPW = 1, 2 or 4 consecutive cars per thread, all in registers).  The
// one-warp kernel above is bound by a single warp's issue rate (about 200
// instructions per step for 200 cars, ~2.3 cycles each: ALU-pipe
// instructions issue every other cycle; 513 ns per step at 16 cars per lane),
// so above 256 cars the ring is spread over the four schedulers instead
// (283 ns at N = 500) and the warps meet once per step: each publishes
// its first car's new position (the leader of the warp behind), its crossing
// count and its velocity sum in a parity-alternating shared-memory slot, one
// barrier, and every thread folds the four counts into W and the draw base
// E exactly as the one-warp kernel does (both candidates of the next base
// precomputed per lane, one shuffle after the count).  EXACT: N a multiple
// of CPW (a thread holds CPW cars or none).
template <typename VT, int CPW, bool EXACT>
__global__ void __launch_bounds__(128, 1) ring_quad_kernel(const RingArgs ra, const uint32_t steps) {
  __shared__ uint32_t apw[256];
  __shared__ __align__(16) uint32_t s_x0[2][4], s_crs[2][4], s_sum[2][4];
  Ctl* ctl = ra.ctl;
  const uint32_t N = ra.n, L = ra.L, vmax = ra.vmax, tp = ra.tp;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint64_t t0 = ctl->t;
  const int b = static_cast<int>(ctl->buf);
  uint32_t* X = xbuf(ra, b);
  VT* V = vbuf_w<VT>(ra, b);
  for (uint32_t i = tid; i < 256; i += 128) apw[i] = c_pow.lin[i];
  uint32_t x[CPW], v[CPW], apA[CPW], apB[CPW];
  uint32_t live = 0;  // bit c: car tid*CPW + c exists
  const uint32_t first = tid * CPW;
  const uint32_t a0 = first < N ? powmod(kA, first) : 1u;
#pragma unroll
  for (int c = 0; c < CPW; ++c) {
    const uint32_t id = first + c;
    const bool ok = id < N;
    live |= ok ? (1u << c) : 0u;
    x[c] = ok ? X[id] : 0u;
    v[c] = ok ? static_cast<uint32_t>(V[id]) : 0u;
    const uint32_t a = mulmod(a0, c_pow.lin[c]);
    apA[c] = a << 1;
    apB[c] = mulmod(a, ra.an_inv) << 1;
  }
  const uint32_t last_tid = (N - 1) / CPW, last_c = (N - 1) % CPW;  // the thread holding car N-1 and its slot
  const uint32_t candw2 = c_pow.lin[lane] << 1;
  const uint32_t candn2 = mulmod(ra.an, c_pow.lin[lane]) << 1;
  uint32_t W = ctl->W, E = ctl->E;
  uint32_t rsum = 0, rc = 0, rW = 0;  // warp 0: batched step records (lane = step mod 32)
  if (lane == 0) s_x0[0][warp] = x[0];
  __syncthreads();
  for (uint32_t st = 0; st < steps; ++st) {
    const uint32_t par = st & 1u;
    const uint32_t bound = N - W;
    const uint32_t nextw = mulmod_x2(candw2, E), nextn = mulmod_x2(candn2, E);
    uint32_t xn = __shfl_down_sync(0xffffffffu, x[0], 1);
    if (lane == 31) xn = s_x0[par][(warp + 1) & 3u];
    const uint32_t x00 = s_x0[par][0];  // leader of car N-1
    uint32_t sum = 0, crs = 0;
    if constexpr (EXACT) {
      if (tid == last_tid) xn = x00;
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        const uint32_t s = mulmod_x2(first + c < bound ? apA[c] : apB[c], E);
        const uint32_t xl = c + 1 < CPW ? x[c + 1 < CPW ? c + 1 : c] : xn;
        uint32_t d = xl - x[c];
        d = min(d, d + L);  // leader past the origin: + L
        const int vc = static_cast<int>(min(min(v[c] + 1, vmax), d - 1));
        int dec;
        asm("mul.hi.s32 %0, %1, 1;" : "=r"(dec) : "r"(static_cast<int>(s - tp)));
        v[c] = static_cast<uint32_t>(max(vc + dec, 0));
        const uint32_t xs = x[c] + v[c];
        x[c] = min(xs, xs - L);
        sum += v[c];
        crs += xs >= L ? 1u : 0u;
      }
      if (!live) sum = crs = 0;  // dead thread
    } else {
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        const uint32_t id = first + c;
        const uint32_t s = mulmod_x2(id < bound ? apA[c] : apB[c], E);
        const uint32_t xl = (tid == last_tid && c == int(last_c)) ? x00 : (c + 1 < CPW ? x[c + 1 < CPW ? c + 1 : c] : xn);
        uint32_t d = xl - x[c];
        d = min(d, d + L);
        const int vc = static_cast<int>(min(min(v[c] + 1, vmax), d - 1));
        const int vnew = max(vc - (s < tp ? 1 : 0), 0);
        const uint32_t xs = x[c] + static_cast<uint32_t>(vnew);
        if ((live >> c) & 1u) {
          v[c] = static_cast<uint32_t>(vnew);
          x[c] = min(xs, xs - L);
          sum += v[c];
          crs += xs >= L ? 1u : 0u;
        }
      }
    }
    crs = __reduce_add_sync(0xffffffffu, crs);
    sum = __reduce_add_sync(0xffffffffu, sum);
    if (lane == 0) {
      s_x0[par ^ 1u][warp] = x[0];
      s_crs[par ^ 1u][warp] = crs;
      s_sum[par ^ 1u][warp] = sum;
    }
    __syncthreads();
    const uint4 c4 = *reinterpret_cast<const uint4*>(s_crs[par ^ 1u]);
    const uint32_t cj = c4.x + c4.y + c4.z + c4.w;
    if (warp == 0) {
      const uint4 s4 = *reinterpret_cast<const uint4*>(s_sum[par ^ 1u]);
      if (lane == (st & 31u)) {
        rsum = s4.x + s4.y + s4.z + s4.w;
        rc = cj;
        rW = W;
      }
      if ((st & 31u) == 31u || st + 1 == steps) {
        if (lane <= (st & 31u)) {
          StepRec* r = ra.rec + ((t0 + (st & ~31u) + lane) % kRecCap);
          r->sumv = rsum;
          r->c = rc;
          r->W = rW;
        }
      }
    }
    uint32_t Wn = W + cj;
    const bool wrap = Wn >= N;
    if (wrap) Wn -= N;
    const uint32_t fast = __shfl_sync(0xffffffffu, wrap ? nextw : nextn, cj & 31u);
    if (cj < 32) {
      E = fast;
    } else {
      const uint32_t ac = cj < 256 ? apw[cj] : powmod(kA, cj);
      E = mulmod_d(E, wrap ? ac : mulmod_d(ra.an, ac));
    }
    W = Wn;
    if (ra.dump) {  // checksum / frame batch: this step's row in rank order
      uint32_t* row = ra.dump + size_t(st) * 2u * N;
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        if ((live >> c) & 1u) {
          uint32_t r = first + c + W;
          if (r >= N) r -= N;
          row[r] = x[c];
          row[N + r] = v[c];
        }
      }
    }
  }
#pragma unroll
  for (int c = 0; c < CPW; ++c) {
    if ((live >> c) & 1u) {
      X[first + c] = x[c];
      V[first + c] = static_cast<VT>(v[c]);
    }
  }
  if (tid == 0) {
    StepRec* nrec = ra.rec + ((t0 + steps) % kRecCap);
    nrec->sumv = 0;
    nrec->c = 0;
    ctl->t = t0 + steps;
    ctl->W = W;
    ctl->E = E;
    ctl->E2 = mulmod_d(E, ra.an_inv);
  }
}

}  // namespace nb200
