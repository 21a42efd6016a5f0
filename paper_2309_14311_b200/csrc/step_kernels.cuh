// step_kernels.cuh -- sm_100a kernels of the NaSch agent step.
//
// One launch = one synchronous time step of the whole ring, i.e. the
// reference's Phase A + Phase B + `omp single` tail of
// Engine::advance_agent (src/engine.cpp:115-181) and step_serial
// (src/model.cpp:42-75), fused:
//
//   per car id (ID order, never rotated; rank(id) = (id + W_t) mod N):
//     gap   = (x[id+1] - x[id] - 1) mod L          (model.hpp:60-65)
//     v     = min(v+1, vmax); v = min(v, gap)       (model.cpp:48-50)
//     s     = minstd output #(t*N + rank + 1)       (counter-based draw)
//     if (s < T_p && v > 0) --v                     (model.cpp:51-53)
//     x'    = (x + v) mod L                          (model.cpp:57-66)
//   reductions: c_t = #cars with x+v >= L  (the reference's wrap count,
//   engine.cpp:138/150-153) and sum(v') (measure, model.cpp:131-142).
//
// The rotation of the wrapped suffix (model.cpp:70-73) is never performed:
// it only shifts every rank by c_t, which W_{t+1} = W_t + c_t absorbs.
//
// HBM layout: x as u32[Npad], v as VT[Npad] (u8 when vmax_eff <= 255),
// ping-pong buffers selected by step parity.  Each thread owns CPT=4
// consecutive cars per tile: one 16-byte x load, one 4-byte (u8) v load,
// the leader of its last car via a warp shuffle (lane 31: one extra 4-byte
// load that hits the line the next warp streams), so HBM sees exactly
// 4+1 bytes read and 4+1 bytes written per car-update.
//
// Step control (W_t, E_t) lives on the device: the LAST block of launch t
// (ticket pattern) folds the step's wrap count into W_{t+1} and the next
// draw base, so consecutive launches (a CUDA graph chain) need no host
// round trip.
#pragma once
#include <cstdint>

#include "minstd.hpp"

namespace nb200 {

struct Ctl {
  unsigned long long t;  // steps completed on the device
  unsigned int W;        // rank offset: rank(id) = (id + W) mod N
  unsigned int E;        // s0 * a^(t*N + 1 + W) mod m: draw of id 0 if 0 < N-W
  unsigned int E2;       // E * a^(-N): draw base for ids >= N - W
  unsigned int ticket;   // last-block-done counter
};

struct StepRec {
  unsigned long long sumv;  // exact sum of velocities after the step
  unsigned int c;           // cars that crossed the origin in the step
  unsigned int W;           // rank offset the step was drawn with
};

constexpr uint32_t kRecCap = 1u << 16;  // device ring of per-step records

struct RingArgs {
  uint32_t* x[2];
  void* v[2];
  uint32_t n;       // cars
  uint32_t L;       // cells (< 2^31)
  uint32_t vmax;    // effective vmax = min(vmax, L-1)
  uint32_t tp;      // deceleration iff draw < tp
  uint32_t s0;      // seeded generator state
  uint32_t an_inv;  // a^(-N) mod m
  uint32_t a1;      // a^(1-N) mod m (step across the rank seam)
  uint32_t g;       // a^(gridDim.x * TILE) mod m (grid-stride advance)
  const uint32_t* blkpow;  // a^(blockIdx.x * TILE)
  const uint32_t* thrpow;  // a^(threadIdx.x * CPT)
  Ctl* ctl;
  StepRec* rec;     // kRecCap ring indexed by t mod kRecCap
};

template <typename VT>
struct VPack;

template <>
struct VPack<uint8_t> {
  using raw = uint32_t;
  static __device__ __forceinline__ raw load(const uint8_t* p) {
    raw r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
  }
  static __device__ __forceinline__ uint32_t get(raw r, int j) { return (r >> (8 * j)) & 0xffu; }
  static __device__ __forceinline__ void put(raw& r, int j, uint32_t v) { r |= v << (8 * j); }
  static __device__ __forceinline__ void store(uint8_t* p, raw r) {
    *reinterpret_cast<uint32_t*>(p) = r;
  }
};

template <>
struct VPack<uint32_t> {
  using raw = uint4;
  static __device__ __forceinline__ raw load(const uint32_t* p) {
    raw r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
  }
  static __device__ __forceinline__ uint32_t get(const raw& r, int j) {
    return j == 0 ? r.x : j == 1 ? r.y : j == 2 ? r.z : r.w;
  }
  static __device__ __forceinline__ void put(raw& r, int j, uint32_t v) {
    if (j == 0) r.x = v; else if (j == 1) r.y = v; else if (j == 2) r.z = v; else r.w = v;
  }
  static __device__ __forceinline__ void store(uint32_t* p, const raw& r) {
    *reinterpret_cast<uint4*>(p) = r;
  }
};

__device__ __forceinline__ uint4 ld_x4(const uint32_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t get4(const uint4& r, int j) {
  return j == 0 ? r.x : j == 1 ? r.y : j == 2 ? r.z : r.w;
}

// One car: returns the new velocity; writes the new position and whether
// it crossed the origin.  All u32: x + v < 2L < 2^32 and xl + (L - x) - 1
// < L, so nothing wraps.
__device__ __forceinline__ uint32_t car_rule(uint32_t x, uint32_t xl, uint32_t v,
                                             uint32_t s, uint32_t L, uint32_t vmax,
                                             uint32_t tp, uint32_t& xnew,
                                             uint32_t& crossed) {
  const uint32_t gap = xl > x ? xl - x - 1 : xl + (L - x) - 1;
  v = min(v + 1, vmax);
  v = min(v, gap);
  v -= (s < tp && v > 0) ? 1u : 0u;
  const uint32_t nx = x + v;
  crossed = nx >= L ? 1u : 0u;
  xnew = crossed ? nx - L : nx;
  return v;
}

template <typename VT, int TPB>
__global__ void __launch_bounds__(TPB) nasch_step_kernel(const RingArgs ra) {
  constexpr int CPT = 4;
  constexpr uint32_t TILE = TPB * CPT;
  const uint32_t N = ra.n;
  const uint64_t t = ra.ctl->t;
  const uint32_t W = ra.ctl->W;
  const uint32_t E = ra.ctl->E;
  const uint32_t E2 = ra.ctl->E2;
  const int par = static_cast<int>(t & 1);
  // select with ternaries: indexing the by-value parameter array with a
  // runtime index would spill it to local memory
  const uint32_t* __restrict__ X = par ? ra.x[1] : ra.x[0];
  const VT* __restrict__ V = static_cast<const VT*>(par ? ra.v[1] : ra.v[0]);
  uint32_t* __restrict__ Xo = par ? ra.x[0] : ra.x[1];
  VT* __restrict__ Vo = static_cast<VT*>(par ? ra.v[0] : ra.v[1]);
  const uint32_t bound = N - W;  // ids >= bound draw from E2 (none when W == 0)
  const uint32_t L = ra.L, vmax = ra.vmax, tp = ra.tp;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t x_head = __ldg(X);  // leader of car N-1 is car 0

  uint32_t P = mulmod(__ldg(ra.blkpow + blockIdx.x), __ldg(ra.thrpow + threadIdx.x));
  unsigned long long sumv = 0;
  uint32_t cross = 0;
  const uint32_t ntiles = (N + TILE - 1) / TILE;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t b = tile * TILE + threadIdx.x * CPT;
    const uint4 xs = ld_x4(X + b);
    const typename VPack<VT>::raw vs = VPack<VT>::load(V + b);
    uint32_t xnext = __shfl_down_sync(0xffffffffu, xs.x, 1);
    if (lane == 31 && b + CPT < N) xnext = __ldg(X + b + CPT);
    uint32_t s = mulmod(P, b < bound ? E : E2);
    P = mulmod(P, ra.g);

    uint4 xo;
    typename VPack<VT>::raw vo{};
    uint32_t tsum = 0, tcross = 0;
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const uint32_t id = b + j;
      if (j > 0) s = mulmod(s, id == bound ? ra.a1 : kA);
      const uint32_t x = get4(xs, j);
      const uint32_t xl = (id + 1 < N) ? (j + 1 < CPT ? get4(xs, j + 1) : xnext) : x_head;
      uint32_t xn, cr;
      const uint32_t vn = car_rule(x, xl, VPack<VT>::get(vs, j), s, L, vmax, tp, xn, cr);
      if (j == 0) xo.x = xn; else if (j == 1) xo.y = xn; else if (j == 2) xo.z = xn; else xo.w = xn;
      VPack<VT>::put(vo, j, vn);
      const bool live = id < N;
      tsum += live ? vn : 0u;
      tcross += live ? cr : 0u;
    }
    *reinterpret_cast<uint4*>(Xo + b) = xo;
    VPack<VT>::store(Vo + b, vo);
    sumv += tsum;
    cross += tcross;
  }

  // Block reduction, then one atomic per block for each of c_t and sum(v).
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sumv += __shfl_xor_sync(0xffffffffu, sumv, o);
    cross += __shfl_xor_sync(0xffffffffu, cross, o);
  }
  __shared__ unsigned long long s_sum[TPB / 32];
  __shared__ uint32_t s_cross[TPB / 32];
  if (lane == 0) {
    s_sum[threadIdx.x / 32] = sumv;
    s_cross[threadIdx.x / 32] = cross;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long bs = 0;
    uint32_t bc = 0;
#pragma unroll
    for (int w = 0; w < TPB / 32; ++w) {
      bs += s_sum[w];
      bc += s_cross[w];
    }
    StepRec* rec = ra.rec + (t % kRecCap);
    if (bs) atomicAdd(&rec->sumv, bs);
    if (bc) atomicAdd(&rec->c, bc);
    __threadfence();
    const uint32_t ticket = atomicAdd(&ra.ctl->ticket, 1u);
    if (ticket == gridDim.x - 1) {
      // Last block: every block's wrap count is in; fold it into the next
      // step's rank offset and draw base (the rotation, model.cpp:70-73).
      __threadfence();
      const uint32_t c = atomicAdd(&rec->c, 0u);
      uint32_t Wn = W + c;  // W < N, c <= N
      if (Wn >= N) Wn -= N;
      const uint32_t En = mulmod(ra.s0, powmod(kA, draw_exponent(t + 1, N, Wn)));
      rec->W = W;
      StepRec* nrec = ra.rec + ((t + 1) % kRecCap);
      nrec->sumv = 0;
      nrec->c = 0;
      nrec->W = Wn;
      ra.ctl->W = Wn;
      ra.ctl->E = En;
      ra.ctl->E2 = mulmod(En, ra.an_inv);
      ra.ctl->t = t + 1;
      ra.ctl->ticket = 0;
    }
  }
}

// x_i = floor(i*L/N), v_i = 0 (model.cpp:30-40), in ID order (= rank order
// at W = 0).
template <typename VT>
__global__ void init_state_kernel(uint32_t* x, VT* v, uint32_t n, uint32_t npad, uint64_t L) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < npad;
       i += (uint64_t)gridDim.x * blockDim.x) {
    x[i] = i < n ? static_cast<uint32_t>(i * L / n) : 0u;
    v[i] = 0;
  }
}

// Exact velocity sum of the current state (observables at step 0).
template <typename VT>
__global__ void sum_velocity_kernel(const VT* v, uint32_t n, unsigned long long* out) {
  unsigned long long s = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    s += v[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// u32 staging -> VT narrowing for set_state (velocities validated on host).
template <typename VT>
__global__ void narrow_velocity_kernel(const uint32_t* src, VT* dst, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = static_cast<VT>(src[i]);
}

}  // namespace nb200
