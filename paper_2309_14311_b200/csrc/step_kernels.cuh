// step_kernels.cuh -- sm_100a kernels of the NaSch agent step.
//
// The reference's time step (step_serial, src/model.cpp:42-75; the OpenMP
// form Engine::advance_agent, src/engine.cpp:101-184) for car i in rank
// order is
//     gap = (x[i+1] - x[i] - 1) mod L            (model.hpp:60-65)
//     v   = min(v+1, vmax); v = min(v, gap)       (model.cpp:48-50)
//     u   = next draw; if (u < p && v > 0) --v   (model.cpp:51-53)
//     x   = (x + v) mod L, then the wrapped suffix rotates to the front.
//
// B200 restatement:
//  * Cars are stored in ID order and never rotated.  The rotation only
//    shifts every rank by the step's wrap count c_t, so
//    rank(id, t) = (id + W_t) mod N with W_{t+1} = W_t + c_t (mod N), and
//    the leader of id is always id+1 (mod N).
//  * The draw of rank r at step t is minstd output #(t*N + r + 1) =
//    s0 * a^(t*N + 1 + W_t) * a^id  [* a^-N when id >= N - W_t]  (mod m):
//    one mulmod per car from per-step bases E_t, E2_t = E_t * a^-N.
//  * u < p  <=>  s < T_p  (integer threshold, minstd.hpp).
//
// Two step kernels:
//  nasch_step_kernel  one launch = one step, streaming (x,v) through HBM
//                     once; the launch's last block folds c_t into W_{t+1}.
//  nasch_tb_kernel    one launch = k <= 16 steps (temporal blocking): each
//                     tile of 2048 consecutive cars (2032 owned + a 16-car
//                     halo ahead) is loaded once into registers, advanced k
//                     steps, and the 2032 owned cars stored once, so HBM
//                     moves ~10/k bytes per car-update.  The k per-step
//                     rank offsets come from the ORIGIN CONE planner, run
//                     by the previous launch's last block: only cars with
//                     x >= L - k*vmax can cross the origin within k steps
//                     (they are the last k*vmax ranks), and simulating them
//                     plus the k cars ahead of the origin for k steps
//                     yields c_t .. c_{t+k-1} exactly.  Every launch
//                     re-counts the crossings and flags any disagreement.
#pragma once
#include <cstdint>

#include "minstd.hpp"

namespace nb200 {

constexpr int kPlanMax = 32;  // steps per temporal-blocked launch (TB kernel; <= its halo)
constexpr int kPlanCap = 32;  // plan capacity of Ctl (the distributed-resident epochs)

struct Ctl {
  unsigned long long t;  // steps completed on the device
  unsigned int W;        // rank offset at step t: rank(id) = (id + W) mod N
  unsigned int buf;      // which ping-pong buffer holds the state at step t
  unsigned int ticket;   // last-block-done counter
  unsigned int err;      // != 0: a launch's crossing count contradicted the plan
  unsigned int E;        // s0 * a^(t*N + 1 + W): draw base of ids < N - W
  unsigned int E2;       // E * a^(-N): draw base of ids >= N - W
  unsigned int kplan;    // steps the plan below covers (temporal blocking)
  unsigned int err_step;
  unsigned int Wk[kPlanCap];   // W_{t+j}
  unsigned int Ek[kPlanCap];   // E_{t+j}
  unsigned int E2k[kPlanCap];  // E2_{t+j}
  unsigned int ck[kPlanCap];   // predicted c_{t+j}
};

struct StepRec {
  unsigned long long sumv;  // exact sum of velocities after the step (this shard's cars)
  unsigned int c;           // cars (of this shard) that crossed the origin in the step
  unsigned int W;           // rank offset the step was drawn with
  unsigned int cplan;       // crossings the origin-cone plan predicted (whole ring)
  unsigned int pad;
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
  uint32_t an;      // a^N mod m
  uint32_t an_inv;  // a^(-N) mod m
  uint32_t a1;      // a^(1-N) mod m (step across the rank seam)
  uint32_t g;       // a^(gridDim.x * tile stride) mod m (grid-stride advance)
  uint32_t kplan;   // temporal-blocking plan length (0: single-step mode)
  uint32_t nl;      // cars stored in this buffer (= n on one GPU; a shard's count otherwise)
  uint32_t gofs;    // global id of local car 0 (0 on one GPU)
  uint32_t agofs;   // a^gofs mod m
  uint32_t sharded; // 1: the halo sits inline after nl and the plan comes from the exchange
  const uint32_t* blkpow;  // a^(blockIdx.x * tile stride)
  const uint32_t* thrpow;  // a^(threadIdx.x * cars per thread)
  Ctl* ctl;
  StepRec* rec;     // kRecCap ring indexed by t mod kRecCap
  // -1 as a launch parameter: ptxas cannot fold it, so x * neg1 + xl stays
  // one IMAD on the FMA pipe instead of an IADD3 on the (busier) ALU pipe.
  uint32_t neg1 = 0xffffffffu;
  // Checksum mode on small rings (engine.cu, GpuRing::Impl::advance): the
  // small-ring kernels write each step's rank-ordered row -- N positions,
  // then N velocities, as u32 -- to dump + 2N * (step within the launch),
  // for one digest over a batch of rows.  nullptr: off.
  uint32_t* dump = nullptr;
  // The row digest (fnv_kernels.cuh) over positions only: the velocity
  // slots are empty (a dump batch is one flat array of u32 values).
  uint32_t fnv_pos_only = 0;
};

// ---- vector access helpers ----------------------------------------------

// Bulk prefetch of [p, p + bytes) into L2 (TMA unit; p and bytes multiples
// of 16): the next tile's state streams in while this tile's steps run.
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_nc_v2(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_nc_u32(const void* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t get4(const uint4& r, int j) {
  return j == 0 ? r.x : j == 1 ? r.y : j == 2 ? r.z : r.w;
}

// Loads/stores CPT consecutive velocities of type VT into u32 registers.
template <typename VT, int CPT>
struct VLanes;

template <>
struct VLanes<uint8_t, 4> {
  static __device__ __forceinline__ void load(const uint8_t* p, uint32_t* v) {
    const uint32_t r = ld_nc_u32(p);
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = (r >> (8 * j)) & 0xffu;
  }
  static __device__ __forceinline__ void store(uint8_t* p, const uint32_t* v) {
    *reinterpret_cast<uint32_t*>(p) = v[0] | (v[1] << 8) | (v[2] << 16) | (v[3] << 24);
  }
};
template <>
struct VLanes<uint8_t, 8> {
  static __device__ __forceinline__ void load(const uint8_t* p, uint32_t* v) {
    const uint2 r = ld_nc_v2(p);
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // one PRMT per byte
      v[j] = __byte_perm(r.x, 0u, 0x4440u | j);
      v[4 + j] = __byte_perm(r.y, 0u, 0x4440u | j);
    }
  }
  static __device__ __forceinline__ uint2 pack(const uint32_t* v) {
    uint2 r;
    r.x = __byte_perm(__byte_perm(v[0], v[1], 0x0040u), __byte_perm(v[2], v[3], 0x0040u), 0x5410u);
    r.y = __byte_perm(__byte_perm(v[4], v[5], 0x0040u), __byte_perm(v[6], v[7], 0x0040u), 0x5410u);
    return r;
  }
  static __device__ __forceinline__ void store(uint8_t* p, const uint32_t* v) {
    *reinterpret_cast<uint2*>(p) = pack(v);
  }
};
template <>
struct VLanes<uint8_t, 16> {
  static __device__ __forceinline__ void load(const uint8_t* p, uint32_t* v) {
    const uint4 r = ld_nc_v4(p);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[j] = __byte_perm(r.x, 0u, 0x4440u | j);
      v[4 + j] = __byte_perm(r.y, 0u, 0x4440u | j);
      v[8 + j] = __byte_perm(r.z, 0u, 0x4440u | j);
      v[12 + j] = __byte_perm(r.w, 0u, 0x4440u | j);
    }
  }
  static __device__ __forceinline__ uint32_t pack4(const uint32_t* v) {
    return __byte_perm(__byte_perm(v[0], v[1], 0x0040u), __byte_perm(v[2], v[3], 0x0040u), 0x5410u);
  }
  static __device__ __forceinline__ void store(uint8_t* p, const uint32_t* v) {
    *reinterpret_cast<uint4*>(p) = make_uint4(pack4(v), pack4(v + 4), pack4(v + 8), pack4(v + 12));
  }
};
template <>
struct VLanes<uint8_t, 32> {
  static __device__ __forceinline__ void load(const uint8_t* p, uint32_t* v) {
    VLanes<uint8_t, 16>::load(p, v);
    VLanes<uint8_t, 16>::load(p + 16, v + 16);
  }
  static __device__ __forceinline__ void store(uint8_t* p, const uint32_t* v) {
    VLanes<uint8_t, 16>::store(p, v);
    VLanes<uint8_t, 16>::store(p + 16, v + 16);
  }
};
template <int CPT>
struct VLanes<uint32_t, CPT> {
  static __device__ __forceinline__ void load(const uint32_t* p, uint32_t* v) {
#pragma unroll
    for (int q = 0; q < CPT / 4; ++q) {
      const uint4 r = ld_nc_v4(p + 4 * q);
#pragma unroll
      for (int j = 0; j < 4; ++j) v[4 * q + j] = get4(r, j);
    }
  }
  static __device__ __forceinline__ void store(uint32_t* p, const uint32_t* v) {
#pragma unroll
    for (int q = 0; q < CPT / 4; ++q)
      *reinterpret_cast<uint4*>(p + 4 * q) = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
};

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

// Sum of small non-negative integers on the FP32 pipe: read as floats, the
// bit patterns of integers below 2^23 are denormals, whose addition
// (without flush-to-zero: PTX add.rn.f32, no .ftz) is exact integer
// addition of the bit patterns.  Moves the temporal-blocked kernel's
// per-step velocity sums off the integer ALU pipe (its binding pipe) onto
// the otherwise idle FP32 lanes.  Valid while every partial sum < 2^23.
__device__ __forceinline__ float fadd_denorm(float a, float b) {
  float r;
  asm("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
template <int CPT>
__device__ __forceinline__ uint32_t vsum_fp32(const uint32_t* v) {
  float t[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) t[c] = __uint_as_float(v[c]);
#pragma unroll
  for (int w = 1; w < CPT; w <<= 1) {
#pragma unroll
    for (int c = 0; c + w < CPT; c += 2 * w) t[c] = fadd_denorm(t[c], t[c + w]);
  }
  return __float_as_uint(t[0]);
}
template <int CPT>
__device__ __forceinline__ uint32_t vsum_imad(const uint32_t* v) {
  uint32_t t[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) t[c] = v[c];
#pragma unroll
  for (int w = 1; w < CPT; w <<= 1) {
#pragma unroll
    for (int c = 0; c + w < CPT; c += 2 * w) {
      uint32_t r;
      asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(t[c]), "r"(1u), "r"(t[c + w]));
      t[c] = r;
    }
  }
  return t[0];
}

// Sum of CPT velocities (u8 lanes: two byte dot-products of the packed
// store words).
template <typename VT, int CPT>
struct VSum {
  static __device__ __forceinline__ uint32_t sum(const uint32_t* v) {
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < CPT; ++c) s += v[c];
    return s;
  }
};
template <>
struct VSum<uint8_t, 8> {
  static __device__ __forceinline__ uint32_t sum(const uint32_t* v) {
    const uint2 p = VLanes<uint8_t, 8>::pack(v);
    return static_cast<uint32_t>(__dp4a(static_cast<int>(p.y), 0x01010101,
                                        __dp4a(static_cast<int>(p.x), 0x01010101, 0)));
  }
};

// Interior car: its leader is strictly ahead without wrapping (xl > x),
// which holds for every car except rank N-1.  Counts a crossing into cnt.
__device__ __forceinline__ uint32_t car_fast(uint32_t x, uint32_t xl, uint32_t v, uint32_t s,
                                             uint32_t L, uint32_t vmax, uint32_t tp,
                                             uint32_t& xnew, uint32_t& cnt) {
  v = min(min(v + 1, vmax), xl - x - 1);
  if (s < tp) v = static_cast<uint32_t>(max(static_cast<int>(v) - 1, 0));
  uint32_t nx = x + v;
  if (nx >= L) {
    nx -= L;
    ++cnt;
  }
  xnew = nx;
  return v;
}

// Any car (the leader may sit behind the origin): gap taken mod L.
__device__ __forceinline__ uint32_t car_any(uint32_t x, uint32_t xl, uint32_t v, uint32_t s,
                                            uint32_t L, uint32_t vmax, uint32_t tp,
                                            uint32_t& xnew, uint32_t& cnt) {
  const uint32_t gap = xl > x ? xl - x - 1 : xl + (L - x) - 1;
  v = min(min(v + 1, vmax), gap);
  if (s < tp) v = static_cast<uint32_t>(max(static_cast<int>(v) - 1, 0));
  uint32_t nx = x + v;
  if (nx >= L) {
    nx -= L;
    ++cnt;
  }
  xnew = nx;
  return v;
}

template <typename VT>
__device__ __forceinline__ const VT* vbuf(const RingArgs& ra, int b) {
  return static_cast<const VT*>(b ? ra.v[1] : ra.v[0]);
}
template <typename VT>
__device__ __forceinline__ VT* vbuf_w(const RingArgs& ra, int b) {
  return static_cast<VT*>(b ? ra.v[1] : ra.v[0]);
}
__device__ __forceinline__ uint32_t* xbuf(const RingArgs& ra, int b) { return b ? ra.x[1] : ra.x[0]; }

// Ticket pattern: returns true in every thread of the block that finished
// last (all other blocks' global writes are visible to it).
__device__ __forceinline__ bool last_block_done(Ctl* ctl) {
  __shared__ uint32_t s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t ticket = atomicAdd(&ctl->ticket, 1u);
    s_last = (ticket == gridDim.x - 1) ? 1u : 0u;
    if (s_last) __threadfence();
  }
  __syncthreads();
  return s_last != 0;
}

// ---- origin cone planner ---------------------------------------------------
//
// Run by ONE block of TPB threads (TPB >= kk*(vmax+1)).  From the state
// (X, V) at step t with rank offset W, simulates cone cars
//   i in [0, M)      : the M = kk*vmax highest ranks (ids just behind the
//                      rank-0 car h = (N - W) mod N) -- every car that can
//                      reach the origin within kk steps is among them;
//   i in [M, M + kk) : ranks 0..kk-1, the leaders those cars need;
// for kk steps with exact draws, and writes W, E, E2 and the crossing count
// of each step into the plan.  Requires L > kk*vmax and N >= M + kk.
// Global id of cone slot i (slots [0, kk*vmax) trail the rank-0 car, the
// next kk lead it).
__device__ __forceinline__ uint32_t cone_slot_id(uint32_t N, uint32_t W, uint32_t M, uint32_t i) {
  const uint32_t h = W == 0 ? 0u : N - W;
  return static_cast<uint32_t>((uint64_t(h) + (N - M) + i) % N);
}

// The cone simulation proper; thread i holds cone slot i's car (x, v).
template <int TPB>
__device__ void cone_simulate(const RingArgs& ra, uint32_t x, uint32_t v, uint64_t t, uint32_t W,
                              uint32_t kk, Ctl* ctl) {
  static_assert(TPB >= 64 && TPB <= 256, "cone block: two warps of setup, slots < 256");
  __shared__ uint32_t s_x[TPB];
  __shared__ uint32_t s_pow[2];
  const uint32_t N = ra.n, L = ra.L, vmax = ra.vmax;
  const uint32_t M = kk * vmax;
  const uint32_t C = M + kk;
  const uint32_t i = threadIdx.x;
  const bool act = i < C;
  const uint32_t id0 = cone_slot_id(N, W, M, 0);
  const uint32_t id = cone_slot_id(N, W, M, i);
  // Warp 0: a^id0; warp 1: a^(t*N + 1 + W).  Slot ids run consecutively
  // from id0 (wrapping past N - 1), so a^id = a^id0 * a^i [* a^-N].
  if (i < 64) {
    const uint32_t r = i < 32 ? powmod_warp(id0) : powmod_warp(draw_exponent(t, N, W));
    if ((i & 31u) == 0) s_pow[i >> 5] = r;
  }
  __syncthreads();
  uint32_t apw = mulmod(s_pow[0], c_pow.lin[i]);
  if (id < id0) apw = mulmod(apw, ra.an_inv);
  if (!act) apw = 1u;
  uint32_t E = mulmod(ra.s0, s_pow[1]);
  uint32_t Wj = W;
  for (uint32_t j = 0; j < kk; ++j) {
    s_x[i] = x;
    __syncthreads();
    const uint32_t xl = (i + 1 < C) ? s_x[i + 1] : x;  // front-most car: unused
    const uint32_t E2 = mulmod(E, ra.an_inv);
    const uint32_t s = mulmod(apw, id < N - Wj ? E : E2);
    uint32_t xn, cr;
    v = car_rule(x, xl, v, s, L, vmax, ra.tp, xn, cr);
    x = xn;
    const uint32_t c = __syncthreads_count(act && i < M && cr);
    if (i == 0) {
      ctl->Wk[j] = Wj;
      ctl->Ek[j] = E;
      ctl->E2k[j] = E2;
      ctl->ck[j] = c;
    }
    uint32_t Wn = Wj + c;
    const bool wrap = Wn >= N;
    if (wrap) Wn -= N;
    // E_{t+j+1} = E_{t+j} * a^(N + W_{j+1} - W_j)
    const uint32_t ac = c_pow.lin[c];  // c <= M < 256
    E = mulmod(E, wrap ? ac : mulmod(ra.an, ac));
    Wj = Wn;
  }
  if (i == 0) {
    ctl->kplan = kk;
    ctl->E = ctl->Ek[0];
    ctl->E2 = ctl->E2k[0];
  }
}

// Plan from the whole ring held by one GPU: cone cars read straight from
// (X, V) with global ids.
template <typename VT, int TPB>
__device__ void cone_plan(const RingArgs& ra, const uint32_t* X, const VT* V, uint64_t t,
                          uint32_t W, uint32_t kk, Ctl* ctl) {
  const uint32_t M = kk * ra.vmax;
  const bool act = threadIdx.x < M + kk;
  const uint32_t id = cone_slot_id(ra.n, W, M, threadIdx.x);
  // .cg loads: the state was just written by other blocks of this launch
  const uint32_t x = act ? __ldcg(X + id) : 0u;
  const uint32_t v = act ? static_cast<uint32_t>(__ldcg(V + id)) : 0u;
  cone_simulate<TPB>(ra, x, v, t, W, kk, ctl);
}

// Plan for the current state (after set_state / construction).
template <typename VT, int TPB>
__global__ void __launch_bounds__(TPB) cone_init_kernel(const RingArgs ra) {
  Ctl* ctl = ra.ctl;
  const int b = static_cast<int>(ctl->buf);
  const uint64_t t = ctl->t;
  const uint32_t W = ctl->W;
  cone_plan<VT, TPB>(ra, xbuf(ra, b), vbuf<VT>(ra, b), t, W, ra.kplan, ctl);
  for (uint32_t j = threadIdx.x; j < ra.kplan; j += TPB) {
    StepRec* r = ra.rec + ((t + j) % kRecCap);
    r->sumv = 0;
    r->c = 0;
  }
}

// ---- single-step streaming kernel -----------------------------------------

template <typename VT, int TPB, int CPT>
__global__ void __launch_bounds__(TPB) nasch_step_kernel(const RingArgs ra) {
  constexpr uint32_t TILE = TPB * CPT;
  const uint32_t N = ra.n;
  Ctl* ctl = ra.ctl;
  const uint64_t t = ctl->t;
  const uint32_t W = ctl->W;
  const uint32_t E = ctl->E;
  const uint32_t E2 = ctl->E2;
  const int b = static_cast<int>(ctl->buf);
  const uint32_t* __restrict__ X = xbuf(ra, b);
  const VT* __restrict__ V = vbuf<VT>(ra, b);
  uint32_t* __restrict__ Xo = xbuf(ra, b ^ 1);
  VT* __restrict__ Vo = vbuf_w<VT>(ra, b ^ 1);
  const uint32_t bound = N - W;  // ids >= bound draw from E2 (none when W == 0)
  const uint32_t L = ra.L, vmax = ra.vmax, tp = ra.tp;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t x_head = __ldg(X);  // leader of car N-1 is car 0

  uint32_t P = mulmod_d(__ldg(ra.blkpow + blockIdx.x), __ldg(ra.thrpow + threadIdx.x));
  unsigned long long sumv = 0;
  uint32_t cross = 0;
  const uint32_t ntiles = (N + TILE - 1) / TILE;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t base = tile * TILE + threadIdx.x * CPT;
    uint32_t x[CPT], v[CPT];
#pragma unroll
    for (int q = 0; q < CPT / 4; ++q) {
      const uint4 r = ld_nc_v4(X + base + 4 * q);
      x[4 * q] = r.x;
      x[4 * q + 1] = r.y;
      x[4 * q + 2] = r.z;
      x[4 * q + 3] = r.w;
    }
    VLanes<VT, CPT>::load(V + base, v);
    uint32_t xnext = __shfl_down_sync(0xffffffffu, x[0], 1);
    if (lane == 31 && base + CPT < N) xnext = __ldg(X + base + CPT);
    const uint32_t ap = P;  // a^base
    P = mulmod_d(P, ra.g);
    uint32_t cnt = 0, tsum = 0;
    if (base + CPT < N && !(base < bound && bound < base + CPT)) {
      // Interior group: all cars live, one draw base, positions increasing
      // except possibly across the last car's leader (the rank seam).
      uint32_t s = mulmod_d(ap, base < bound ? E : E2);
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        if (c) s = mulmod_d(s, kA);
        if (c + 1 < CPT) {
          v[c] = car_fast(x[c], x[c + 1], v[c], s, L, vmax, tp, x[c], cnt);
        } else {
          v[c] = car_any(x[c], xnext, v[c], s, L, vmax, tp, x[c], cnt);
        }
      }
      tsum = VSum<VT, CPT>::sum(v);
    } else {
      uint32_t s = mulmod_d(ap, base < bound ? E : E2);
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const uint32_t id = base + c;
        if (c) s = mulmod_d(s, id == bound ? ra.a1 : kA);
        const uint32_t xl = (id + 1 < N) ? (c + 1 < CPT ? x[c + 1] : xnext) : x_head;
        uint32_t cc = 0;
        v[c] = car_any(x[c], xl, v[c], s, L, vmax, tp, x[c], cc);
        const bool live = id < N;
        tsum += live ? v[c] : 0u;
        cnt += live ? cc : 0u;
      }
    }
#pragma unroll
    for (int q = 0; q < CPT / 4; ++q)
      *reinterpret_cast<uint4*>(Xo + base + 4 * q) =
          make_uint4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
    VLanes<VT, CPT>::store(Vo + base, v);
    sumv += tsum;
    cross += cnt;
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
  StepRec* rec = ra.rec + (t % kRecCap);
  if (threadIdx.x == 0) {
    unsigned long long bs = 0;
    uint32_t bc = 0;
#pragma unroll
    for (int w = 0; w < TPB / 32; ++w) {
      bs += s_sum[w];
      bc += s_cross[w];
    }
    if (bs) atomicAdd(&rec->sumv, bs);
    if (bc) atomicAdd(&rec->c, bc);
  }
  if (last_block_done(ctl) && threadIdx.x == 0) {
    // Every block's wrap count is in: fold it into the next step's rank
    // offset and draw base (the rotation, model.cpp:70-73).
    const uint32_t c = atomicAdd(&rec->c, 0u);
    uint32_t Wn = W + c;  // W < N, c <= N
    const bool wrap = Wn >= N;
    if (wrap) Wn -= N;
    // exponent t*N + 1 + W grows by N + c (- N when W wraps)
    const uint32_t ac = c < 256 ? c_pow.lin[c] : powmod(kA, c);
    const uint32_t En = mulmod(E, wrap ? ac : mulmod(ra.an, ac));
    rec->W = W;
    StepRec* nrec = ra.rec + ((t + 1) % kRecCap);
    nrec->sumv = 0;
    nrec->c = 0;
    nrec->W = Wn;
    ctl->W = Wn;
    ctl->E = En;
    ctl->E2 = mulmod(En, ra.an_inv);
    ctl->t = t + 1;
    ctl->buf = static_cast<unsigned int>(b ^ 1);
    ctl->ticket = 0;
  }
}

// The temporal-blocked kernel lives in tb_kernel.cuh.

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

// set_state32's position rules on the device (the positions are uploaded
// straight from the caller's page-locked array, so the host never reads
// them): the first violation as 4 i + (rule - 1), rule 1 x >= L, rule 2 not
// strictly increasing (host: src/model.cpp / acceptance.cpp:118-123 order).
static __global__ void validate_positions_kernel(const uint32_t* __restrict__ x, uint32_t n, uint32_t L,
                                          unsigned long long* code) {
  unsigned long long best = ~0ull;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t xi = __ldg(x + i);
    if (xi >= L) best = min(best, 4ull * i);
    else if (i && __ldg(x + i - 1) >= xi) best = min(best, 4ull * i + 1);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(code, best);
}

// The space-time raster row of a frame (src/io.cpp:186-216: a P5 row of L
// pixels, 0 where a car stands, 255 elsewhere), from the ID-ordered
// positions: the row was set to 255 first (cudaMemsetAsync).
static __global__ void raster_kernel(const uint32_t* __restrict__ x, uint32_t n, uint8_t* row) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) row[__ldg(x + i)] = 0;
}

// The current state's rank-ordered row into a dump slot (2N u32 values:
// positions, then velocities), for checksum batches of rings stepped by
// the one-step kernel.
template <typename VT>
__global__ void dump_row_kernel(const RingArgs ra, uint32_t* row) {
  const Ctl* ctl = ra.ctl;
  const uint32_t N = ra.n, W = ctl->W;
  const int b = static_cast<int>(ctl->buf);
  const uint32_t* X = xbuf(ra, b);
  const VT* V = vbuf<VT>(ra, b);
  for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id < N; id += gridDim.x * blockDim.x) {
    uint32_t r = id + W;
    if (r >= N) r -= N;
    row[r] = __ldg(X + id);
    row[N + r] = static_cast<uint32_t>(__ldg(V + id));
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

}  // namespace nb200
