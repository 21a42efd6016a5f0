// ensemble.cu -- GpuEnsemble: many independent rings, each resident in one
// SM's shared memory for a whole launch (see ensemble.hpp).
//
// Kernel: persistent, one 1024-thread CTA per SM with ~227 KB of shared
// memory, pulling rings from an atomic queue in decreasing-N order (longest
// processing time first).  A ring's cars are packed as x | v << bx into one
// u32 per car (bx = bits of L-1; needs bx + bits(vmax) <= 32), so a 57k-car
// ring fits; each thread owns an odd-sized run of consecutive cars (odd
// stride => conflict-free shared-memory banks).  Per step: read the leader
// of the run's last car, barrier, update the run in place (each car reads
// its own word and its leader's old word before overwriting its own),
// warp-reduce the crossing count and velocity sum into per-warp slots,
// barrier.  Every warp then folds the 32 crossing slots into its own copy of
// W and the draw base E (c <= vmax <= 255, so a^c is a table lookup) --
// the rank/draw bookkeeping of the single-ring kernels (step_kernels.cuh)
// with no global round trip.  Rings that do not fit run on a GpuRing each.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine.hpp"
#include "host_simd.hpp"
#include "ensemble.hpp"
#include "minstd.hpp"
#include "tb_config.hpp"
#include "ensemble_tb.cuh"
#include "step_kernels.cuh"

namespace nb200 {

namespace {

void check_e(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  }
}
#define CKE(call) check_e((call), #call)

constexpr int kEnsTPB = 1024;
// a^c table, crossing/velocity slots, scalars, lead slots [2][TPB]
constexpr int kEnsHeaderWords = 256 + 64 + 64 + 16 + 2 * kEnsTPB;

struct RingDesc {
  unsigned long long off;         // first car of the ring in X / V
  unsigned long long t;           // steps done
  unsigned long long steps;       // configured total
  unsigned long long sumv_total;  // sum over completed steps of sum(v)
  uint32_t n, L, vmax, tp, s0, an, an_inv, a1;
  uint32_t W, E, bx, last_sumv;
};

__device__ __forceinline__ uint32_t warp_sum(uint32_t v) { return __reduce_add_sync(0xffffffffu, v); }

template <int TPB>
__global__ void __launch_bounds__(TPB, 1)
    ensemble_kernel(RingDesc* __restrict__ rings, const uint32_t* __restrict__ order, uint32_t nrings,
                    unsigned long long steps, uint32_t* counter, uint32_t* __restrict__ X,
                    uint8_t* __restrict__ V) {
  extern __shared__ uint32_t sm[];
  uint32_t* apw = sm;               // a^c, c < 256
  uint32_t* slot_c = sm + 256;      // [2][32] crossing counts per warp
  uint32_t* slot_v = slot_c + 64;   // [2][32] velocity sums per warp
  uint32_t* sc = slot_v + 64;       // scalars
  uint32_t* leadslot = sc + 16;     // [2][TPB] first position of each thread's run
  uint32_t* packed = sm + kEnsHeaderWords;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  if (tid < 256) apw[tid] = powmod(kA, tid);

  for (;;) {
    __syncthreads();  // previous ring fully written back; sc reusable
    if (tid == 0) sc[0] = atomicAdd(counter, 1u);
    __syncthreads();
    const uint32_t qi = sc[0];
    if (qi >= nrings) break;
    const uint32_t r = order[qi];
    const RingDesc d = rings[r];
    const unsigned long long remain = d.steps - d.t;
    const unsigned long long todo = steps < remain ? steps : remain;
    if (todo == 0) continue;
    const uint32_t N = d.n, L = d.L, vmax = d.vmax, tp = d.tp, bx = d.bx;
    const uint32_t xmask = (1u << bx) - 1u;
    for (uint32_t i = tid; i < N; i += TPB)
      packed[i] = X[d.off + i] | (static_cast<uint32_t>(V[d.off + i]) << bx);
    uint32_t cpt = (N + TPB - 1) / TPB;
    cpt |= 1u;  // odd stride: conflict-free banks
    const uint32_t first = tid * cpt;
    const uint32_t cnt = first < N ? min(cpt, N - first) : 0u;
    // the car after this run is the first car of the next thread's run
    const uint32_t next_tid = (first + cnt >= N) ? 0u : tid + 1;
    const uint32_t ap0 = cnt ? powmod(kA, first) : 1u;
    uint32_t W = d.W, E = d.E;
    unsigned long long total = 0;  // meaningful in warp 0 lane 0
    uint32_t last = d.last_sumv;
    __syncthreads();
    // One barrier per step: each thread publishes its run's first position
    // (state st) in a slot alternating with the step parity, so the thread
    // behind reads its leader there and nobody reads a run being updated.
    for (unsigned long long st = 0; st <= todo; ++st) {
      const uint32_t par = static_cast<uint32_t>(st & 1);
      if (st < todo && cnt) leadslot[par * TPB + tid] = packed[first] & xmask;
      __syncthreads();
      if (st > 0) {
        // fold the previous step's crossings into W and E (every warp)
        const uint32_t p = par ^ 1u;
        const uint32_t c = warp_sum(slot_c[p * 32 + lane]);
        const uint32_t sv = warp_sum(slot_v[p * 32 + lane]);
        total += sv;
        last = sv;
        uint32_t Wn = W + c;
        const bool wrap = Wn >= N;
        if (wrap) Wn -= N;
        E = mulmod_d(E, wrap ? apw[c] : mulmod_d(d.an, apw[c]));
        W = Wn;
      }
      if (st == todo) break;
      const uint32_t E2 = mulmod_d(E, d.an_inv);
      const uint32_t bound = N - W;
      const uint32_t lead = cnt ? leadslot[par * TPB + next_tid] : 0u;
      uint32_t crs = 0, sum = 0;
      // Plain run: the rank seam is neither inside it nor at its last car's
      // leader, and its farthest car cannot reach L this step -- positions
      // increase along the run, no mod L, one draw base.
      const bool plain = cnt && !(first < bound && bound <= first + cnt) &&
                         (packed[first + cnt - 1] & xmask) + vmax < L;
      if (plain) {
        uint32_t s = mulmod_d(ap0, first < bound ? E : E2);
        uint32_t cur = packed[first];
#pragma unroll 2
        for (uint32_t c = 0; c < cnt; ++c) {
          const uint32_t id = first + c;
          if (c) s = mulmod_x2(2u * kA, s);
          const uint32_t nxt = (c + 1 < cnt) ? packed[id + 1] : lead;
          const uint32_t x = cur & xmask;
          uint32_t vn = min(min((cur >> bx) + 1, vmax), (nxt & xmask) - x - 1);
          if (s < tp) vn = static_cast<uint32_t>(max(static_cast<int>(vn) - 1, 0));
          packed[id] = (x + vn) | (vn << bx);
          sum += vn;
          cur = nxt;
        }
      } else if (cnt) {
        uint32_t s = mulmod_d(ap0, first < bound ? E : E2);
        uint32_t cur = packed[first];
        for (uint32_t c = 0; c < cnt; ++c) {
          const uint32_t id = first + c;
          if (c) s = mulmod_d(s, id == bound ? d.a1 : kA);
          const uint32_t nxt = (c + 1 < cnt) ? packed[id + 1] : lead;
          uint32_t xn;
          const uint32_t vn = car_any(cur & xmask, nxt & xmask, cur >> bx, s, L, vmax, tp, xn, crs);
          packed[id] = xn | (vn << bx);
          sum += vn;
          cur = nxt;
        }
      }
      crs = warp_sum(crs);
      sum = warp_sum(sum);
      if (lane == 0) {
        slot_c[par * 32 + warp] = crs;
        slot_v[par * 32 + warp] = sum;
      }
    }
    for (uint32_t i = tid; i < N; i += TPB) {
      const uint32_t w = packed[i];
      X[d.off + i] = w & xmask;
      V[d.off + i] = static_cast<uint8_t>(w >> bx);
    }
    if (tid == 0) {
      rings[r].t = d.t + todo;
      rings[r].W = W;
      rings[r].E = E;
      rings[r].sumv_total = d.sumv_total + total;
      rings[r].last_sumv = last;
    }
  }
}

// init_state (model.cpp:30-40) for every resident ring: block per ring.
__global__ void ensemble_init_kernel(const RingDesc* __restrict__ rings, uint32_t nrings,
                                     uint32_t* __restrict__ X, uint8_t* __restrict__ V) {
  for (uint32_t r = blockIdx.x; r < nrings; r += gridDim.x) {
    const RingDesc d = rings[r];
    for (uint32_t i = threadIdx.x; i < d.n; i += blockDim.x) {
      X[d.off + i] = static_cast<uint32_t>(uint64_t(i) * d.L / d.n);
      V[d.off + i] = 0;
    }
  }
}

// init_state (model.cpp:30-40), tiled layout.
__global__ void ens_tiled_init_kernel(const EnsRing* __restrict__ rings, uint32_t nrings,
                                      uint32_t* __restrict__ X, uint8_t* __restrict__ V) {
  for (uint32_t r = blockIdx.x; r < nrings; r += gridDim.x) {
    const EnsRing d = rings[r];
    for (uint32_t i = threadIdx.x; i < d.n; i += blockDim.x) {
      X[d.off + i] = static_cast<uint32_t>(uint64_t(i) * d.L / d.n);
      V[d.off + i] = 0;
    }
  }
}

uint32_t bits_for(uint64_t max_value) {
  uint32_t b = 0;
  while (b < 32 && (uint64_t(1) << b) <= max_value) ++b;
  return b;
}

}  // namespace

// set_state_all32 with page-locked positions: the concatenated input goes up
// in one DMA (velocities narrowed to u8 on the host) and one block per ring
// scatters its cars into the tiled layout's idle buffer (buf ^ 1), checks
// the position rules (first violation as 4 (global index) + rule - 1, by
// atomicMin) and sums the velocities; ens_commit_kernel then makes the idle
// buffer current, only if no rule failed, so a rejected state leaves every
// ring as it was.
__global__ void __launch_bounds__(256) ens_load_kernel(const EnsArgs ea, const unsigned long long* __restrict__ start,
                                                       const uint32_t* __restrict__ in_x,
                                                       const uint8_t* __restrict__ in_v, uint32_t* sums,
                                                       unsigned long long* code) {
  __shared__ uint32_t s_sum[8];
  const uint32_t r = blockIdx.x;
  const EnsRing R = ea.rings[r];
  const unsigned long long g0 = start[r];
  uint32_t* X = ea.X[R.buf ^ 1u] + R.off;
  uint8_t* V = ea.V[R.buf ^ 1u] + R.off;
  unsigned long long best = ~0ull;
  uint32_t sum = 0;
  for (uint32_t i = threadIdx.x; i < R.n; i += blockDim.x) {
    const uint32_t xi = __ldg(in_x + g0 + i);
    const uint8_t vi = __ldg(in_v + g0 + i);
    X[i] = xi;
    V[i] = vi;
    sum += vi;
    if (xi >= R.L) best = min(best, 4ull * (g0 + i));
    else if (i && __ldg(in_x + g0 + i - 1) >= xi) best = min(best, 4ull * (g0 + i) + 1);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s_sum[threadIdx.x / 32] = sum;
    if (best != ~0ull) atomicMin(code, best);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < 8; ++w) t += s_sum[w];
    sums[r] = t;
  }
}

__global__ void ens_commit_kernel(const EnsArgs ea, const uint32_t* sums, const unsigned long long* code,
                                  unsigned long long host_code) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= ea.nrings || *code != ~0ull || host_code != ~0ull) return;
  EnsRing& R = ea.rings[r];
  R.buf ^= 1u;
  R.W = 0;
  R.k = 0;
  R.last_sumv = sums[r];
}

struct GpuEnsemble::Impl {
  std::vector<SimParams> params;
  int device = 0;
  cudaStream_t stream = nullptr;
  std::vector<int> slot;                    // ring -> resident index or -1
  std::vector<RingDesc> desc;               // resident descriptors (host copy)
  std::vector<std::unique_ptr<GpuRing>> overflow;  // ring -> engine if not resident
  std::vector<uint32_t> order;              // resident indices by decreasing N
  RingDesc* d_desc = nullptr;
  uint32_t* d_order = nullptr;
  uint32_t* d_counter = nullptr;
  uint32_t* X = nullptr;
  uint8_t* V = nullptr;
  RingDesc* h_desc = nullptr;  // pinned mirror
  int grid = 1;
  size_t smem = 0;
  size_t cap_cars = 0;
  uint64_t launches = 0;
  bool dirty = false;  // device descriptors newer than host mirror
  ~Impl();

  // Tiled mode (ensemble_tb.cuh): every ring in warp tiles, K steps per
  // launch; used when every ring is eligible (NASCH_B200_ENS_TILED=0 off).
  bool tiled = false;
  std::vector<EnsRing> trings;
  EnsArgs ea{};
  EnsRing* h_trings = nullptr;
  int tgrid = 1;
  uint32_t K = kEtK;  // steps per tiled launch (<= kEtK, cone <= 512 cars)
  // pinned staging in the tiled layout (set_state_all32)
  size_t stage_cars = 0;
  uint32_t* h_stage_x = nullptr;
  uint8_t* h_stage_v = nullptr;
  // set_state_all32 with page-locked positions (ens_load_kernel)
  uint32_t* d_in_x = nullptr;
  uint8_t* d_in_v = nullptr;
  unsigned long long* d_start = nullptr;
  uint32_t* d_sums = nullptr;
  unsigned long long* d_code = nullptr;
  unsigned long long* h_code = nullptr;

  void tpull() {
    if (!dirty) return;
    CKE(cudaMemcpyAsync(h_trings, ea.rings, trings.size() * sizeof(EnsRing), cudaMemcpyDeviceToHost, stream));
    CKE(cudaStreamSynchronize(stream));
    std::memcpy(trings.data(), h_trings, trings.size() * sizeof(EnsRing));
    dirty = false;
    for (const EnsRing& r : trings)
      if (r.err) throw std::runtime_error("ensemble: origin-cone plan contradicted (engine state is invalid)");
  }

  void tpush() {
    std::memcpy(h_trings, trings.data(), trings.size() * sizeof(EnsRing));
    CKE(cudaMemcpyAsync(ea.rings, h_trings, trings.size() * sizeof(EnsRing), cudaMemcpyHostToDevice, stream));
    CKE(cudaStreamSynchronize(stream));
  }

  void tlaunch(uint64_t steps) {
    const int pgrid = static_cast<int>((trings.size() + 7) / 8);
    for (uint64_t left = steps; left > 0;) {
      const uint32_t kq = static_cast<uint32_t>(std::min<uint64_t>(left, K));
      ens_plan_kernel<<<pgrid, 256, 0, stream>>>(ea, kq);
      ens_tb_kernel<kEtTPB><<<tgrid, kEtTPB, 0, stream>>>(ea);
      CKE(cudaGetLastError());
      launches += 2;
      left -= kq;
    }
    ens_plan_kernel<<<pgrid, 256, 0, stream>>>(ea, 0u);  // fold the last launch
    CKE(cudaGetLastError());
    ++launches;
    dirty = true;
  }

  void pull() {
    if (!dirty || desc.empty()) return;
    CKE(cudaMemcpyAsync(h_desc, d_desc, desc.size() * sizeof(RingDesc), cudaMemcpyDeviceToHost, stream));
    CKE(cudaStreamSynchronize(stream));
    std::memcpy(desc.data(), h_desc, desc.size() * sizeof(RingDesc));
    dirty = false;
  }

  void push() {
    std::memcpy(h_desc, desc.data(), desc.size() * sizeof(RingDesc));
    CKE(cudaMemcpyAsync(d_desc, h_desc, desc.size() * sizeof(RingDesc), cudaMemcpyHostToDevice, stream));
    CKE(cudaStreamSynchronize(stream));
  }

  void launch(uint64_t steps) {
    if (desc.empty()) return;
    CKE(cudaMemsetAsync(d_counter, 0, sizeof(uint32_t), stream));
    ensemble_kernel<kEnsTPB><<<grid, kEnsTPB, smem, stream>>>(
        d_desc, d_order, static_cast<uint32_t>(desc.size()), steps, d_counter, X, V);
    CKE(cudaGetLastError());
    ++launches;
    dirty = true;
  }
};

GpuEnsemble::GpuEnsemble(const std::vector<SimParams>& rings) : impl_(new Impl) {
  Impl& d = *impl_;
  int ndev = 0;
  const cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    throw std::runtime_error(std::string("no CUDA device available for the B200 engine (") +
                             cudaGetErrorString(e) + ")");
  }
  if (rings.empty()) throw std::invalid_argument("ensemble needs at least one ring");
  for (const SimParams& p : rings) {
    p.validate();
    if (p.road_length > 2147483647ull)
      throw std::invalid_argument("length above 2^31-1 is not supported by the B200 engine");
  }
  CKE(cudaGetDevice(&d.device));
  d.params = rings;
  CKE(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
  int max_optin = 0, sms = 0;
  CKE(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, d.device));
  CKE(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d.device));
  d.cap_cars = static_cast<size_t>(max_optin) / 4 - kEnsHeaderWords;

  // Tiled mode when every ring fits the warp-tile step and its cone plan.
  bool all_tiled = std::getenv("NASCH_B200_ENS_TILED") == nullptr ||
                   std::string(std::getenv("NASCH_B200_ENS_TILED")) != "0";
  // Steps per launch K <= the halo, shared by all rings: the planner warp
  // simulates K (vmax + 1) <= 512 cone cars, and every ring must hold a
  // K-step cone (N >= K (vmax + 1), L > K vmax).  Tiled when K >= 8.
  for (const SimParams& p : rings) {
    const uint64_t vm = std::min<uint64_t>(p.v_max, p.road_length - 1);
    all_tiled = all_tiled && vm <= 31;
    uint64_t k = std::min<uint64_t>(512u / (vm + 1), p.car_count / (vm + 1));
    if (vm) k = std::min<uint64_t>(k, (p.road_length - 1) / vm);
    d.K = static_cast<uint32_t>(std::min<uint64_t>(d.K, k));
  }
  all_tiled = all_tiled && d.K >= 8;
  d.K = std::max<uint32_t>(d.K, 1u);
  if (all_tiled) {
    d.tiled = true;
    uint64_t total = 0;
    std::vector<EnsTile> tiles;
    for (size_t r = 0; r < rings.size(); ++r) {
      const SimParams& p = rings[r];
      EnsRing er{};
      er.off = total;
      er.steps = p.steps;
      er.n = static_cast<uint32_t>(p.car_count);
      er.L = static_cast<uint32_t>(p.road_length);
      er.vmax = static_cast<uint32_t>(std::min<uint64_t>(p.v_max, p.road_length - 1));
      er.tp = deceleration_threshold(p.p);
      er.s0 = seeded(p.seed);
      er.an = powmod(kA, er.n);
      er.an_inv = powmod(kA, kOrder - (er.n % kOrder));
      d.trings.push_back(er);
      for (uint32_t b = 0; b < er.n; b += kEtStore)
        tiles.push_back(EnsTile{static_cast<uint32_t>(r), b, powmod(kA, b), 0u});
      total += (er.n + 15) / 16 * 16;  // 16-car aligned rings: vector loads
    }
    const size_t pad = total + kEtLoad + 16;
    // pinned staging for set_state_all32 in the tiled layout, pinned once
    // here (pinning ~0.5 GB costs ~0.1 s: not per call)
    d.stage_cars = total;
    CKE(cudaMallocHost(&d.h_stage_x, total * 4));
    CKE(cudaMallocHost(&d.h_stage_v, total));
    {
      std::vector<unsigned long long> st(rings.size() + 1, 0);
      for (size_t r = 0; r < rings.size(); ++r) st[r + 1] = st[r] + rings[r].car_count;
      CKE(cudaMalloc(&d.d_in_x, std::max<size_t>(1, st.back()) * 4));
      CKE(cudaMalloc(&d.d_in_v, std::max<size_t>(1, st.back())));
      CKE(cudaMalloc(&d.d_start, st.size() * sizeof(unsigned long long)));
      CKE(cudaMemcpy(d.d_start, st.data(), st.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
      CKE(cudaMalloc(&d.d_sums, rings.size() * 4));
      CKE(cudaMalloc(&d.d_code, sizeof(unsigned long long)));
      CKE(cudaMallocHost(&d.h_code, sizeof(unsigned long long)));
    }
    std::memset(d.h_stage_x, 0, total * 4);
    std::memset(d.h_stage_v, 0, total);
    for (int b = 0; b < 2; ++b) {
      CKE(cudaMalloc(&d.ea.X[b], pad * 4));
      CKE(cudaMalloc(&d.ea.V[b], pad));
      CKE(cudaMemset(d.ea.X[b], 0, pad * 4));
      CKE(cudaMemset(d.ea.V[b], 0, pad));
    }
    CKE(cudaMalloc(&d.ea.rings, d.trings.size() * sizeof(EnsRing)));
    CKE(cudaMallocHost(&d.h_trings, d.trings.size() * sizeof(EnsRing)));
    CKE(cudaMalloc(&d.ea.plans, d.trings.size() * sizeof(Ctl)));
    CKE(cudaMalloc(&d.ea.counts, d.trings.size() * sizeof(EnsCount)));
    CKE(cudaMemset(d.ea.counts, 0, d.trings.size() * sizeof(EnsCount)));
    EnsTile* dt = nullptr;
    CKE(cudaMalloc(&dt, tiles.size() * sizeof(EnsTile)));
    CKE(cudaMemcpy(dt, tiles.data(), tiles.size() * sizeof(EnsTile), cudaMemcpyHostToDevice));
    d.ea.tiles = dt;
    std::vector<uint32_t> thr(32);
    for (uint32_t l = 0; l < 32; ++l) thr[l] = powmod(kA, uint64_t(l) * kEtCPT);
    uint32_t* dthr = nullptr;
    CKE(cudaMalloc(&dthr, 32 * 4));
    CKE(cudaMemcpy(dthr, thr.data(), 32 * 4, cudaMemcpyHostToDevice));
    d.ea.thrpow = dthr;
    d.ea.nrings = static_cast<uint32_t>(d.trings.size());
    d.ea.ntiles = static_cast<uint32_t>(tiles.size());
    d.ea.neg1 = 0xffffffffu;
    int per_sm = 0;
    CKE(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ens_tb_kernel<kEtTPB>, kEtTPB, 0));
    const uint64_t blocks_needed = (tiles.size() + kEtTPB / 32 - 1) / (kEtTPB / 32);
    const char* we = std::getenv("NASCH_B200_WAVES");
    const long waves = std::max<long>(1, we && *we ? std::strtol(we, nullptr, 10) : kTbWaves);
    d.tgrid = static_cast<int>(std::max<uint64_t>(
        1, std::min<uint64_t>(blocks_needed, uint64_t(sms) * std::max(per_sm, 1) * uint64_t(waves))));
    d.tpush();
    ens_tiled_init_kernel<<<static_cast<int>(std::min<size_t>(d.trings.size(), 4096)), 256, 0, d.stream>>>(
        d.ea.rings, d.ea.nrings, d.ea.X[0], d.ea.V[0]);
    CKE(cudaGetLastError());
    CKE(cudaStreamSynchronize(d.stream));
    d.slot.assign(rings.size(), 0);
    d.overflow.resize(rings.size());
    return;
  }

  // Which rings are resident, and their packing.
  d.slot.assign(rings.size(), -1);
  d.overflow.resize(rings.size());
  uint64_t total_cars = 0;
  size_t max_cars = 0;
  for (size_t r = 0; r < rings.size(); ++r) {
    const SimParams& p = rings[r];
    const uint64_t vmax_eff = std::min<uint64_t>(p.v_max, p.road_length - 1);
    const uint32_t bx = std::max<uint32_t>(1, bits_for(p.road_length - 1));
    const bool fits = p.car_count <= d.cap_cars && vmax_eff <= 255 &&
                      bx + bits_for(vmax_eff) <= 32;
    if (!fits) continue;
    RingDesc rd{};
    rd.off = total_cars;
    rd.t = 0;
    rd.steps = p.steps;
    rd.n = static_cast<uint32_t>(p.car_count);
    rd.L = static_cast<uint32_t>(p.road_length);
    rd.vmax = static_cast<uint32_t>(vmax_eff);
    rd.tp = deceleration_threshold(p.p);
    rd.s0 = seeded(p.seed);
    rd.an = powmod(kA, rd.n);
    rd.an_inv = powmod(kA, kOrder - (rd.n % kOrder));
    rd.a1 = powmod(kA, (1 + kOrder - (rd.n % kOrder)) % kOrder);
    rd.W = 0;
    rd.E = mulmod(rd.s0, powmod(kA, draw_exponent(0, rd.n, 0)));
    rd.bx = bx;
    d.slot[r] = static_cast<int>(d.desc.size());
    d.desc.push_back(rd);
    total_cars += rd.n;
    max_cars = std::max<size_t>(max_cars, rd.n);
  }
  for (size_t r = 0; r < rings.size(); ++r) {
    if (d.slot[r] < 0) {
      SimParams p = rings[r];
      p.output_mode = OutputMode::none;
      d.overflow[r].reset(new GpuRing(p));
      d.overflow[r]->set_checksum(false);
    }
  }
  if (!d.desc.empty()) {
    d.order.resize(d.desc.size());
    std::iota(d.order.begin(), d.order.end(), 0u);
    std::stable_sort(d.order.begin(), d.order.end(),
                     [&](uint32_t a, uint32_t b) { return d.desc[a].n > d.desc[b].n; });
    CKE(cudaMalloc(&d.X, total_cars * 4 + 16));
    CKE(cudaMalloc(&d.V, total_cars + 16));
    CKE(cudaMalloc(&d.d_desc, d.desc.size() * sizeof(RingDesc)));
    CKE(cudaMallocHost(&d.h_desc, d.desc.size() * sizeof(RingDesc)));
    CKE(cudaMalloc(&d.d_order, d.order.size() * 4));
    CKE(cudaMalloc(&d.d_counter, 4));
    CKE(cudaMemcpy(d.d_order, d.order.data(), d.order.size() * 4, cudaMemcpyHostToDevice));
    d.push();
    d.smem = (kEnsHeaderWords + max_cars) * 4;
    CKE(cudaFuncSetAttribute(ensemble_kernel<kEnsTPB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(d.smem)));
    int per_sm = 0;
    CKE(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ensemble_kernel<kEnsTPB>, kEnsTPB, d.smem));
    d.grid = static_cast<int>(std::min<size_t>(d.desc.size(), size_t(sms) * std::max(per_sm, 1)));
    ensemble_init_kernel<<<static_cast<int>(std::min<size_t>(d.desc.size(), 4096)), 256, 0, d.stream>>>(
        d.d_desc, static_cast<uint32_t>(d.desc.size()), d.X, d.V);
    CKE(cudaGetLastError());
    CKE(cudaStreamSynchronize(d.stream));
  }
}

// Released by Impl's destructor: nothing leaks if construction throws.
GpuEnsemble::Impl::~Impl() {
  cudaSetDevice(device);
  if (stream) cudaStreamSynchronize(stream);
  cudaFree(X);
  cudaFree(V);
  cudaFree(d_desc);
  cudaFree(d_order);
  cudaFree(d_counter);
  cudaFreeHost(h_desc);
  for (int b = 0; b < 2; ++b) {
    cudaFree(ea.X[b]);
    cudaFree(ea.V[b]);
  }
  cudaFree(ea.rings);
  cudaFree(ea.plans);
  cudaFree(ea.counts);
  cudaFree(const_cast<EnsTile*>(ea.tiles));
  cudaFree(const_cast<uint32_t*>(ea.thrpow));
  cudaFreeHost(h_trings);
  cudaFreeHost(h_stage_x);
  cudaFreeHost(h_stage_v);
  cudaFree(d_in_x);
  cudaFree(d_in_v);
  cudaFree(d_start);
  cudaFree(d_sums);
  cudaFree(d_code);
  cudaFreeHost(h_code);
  if (stream) cudaStreamDestroy(stream);
}

GpuEnsemble::~GpuEnsemble() = default;

size_t GpuEnsemble::size() const { return impl_->params.size(); }
size_t GpuEnsemble::resident_capacity_cars() const { return impl_->cap_cars; }
void* GpuEnsemble::cuda_stream() const { return impl_->stream; }

uint64_t GpuEnsemble::kernel_launches() const {
  uint64_t n = impl_->launches;
  for (const auto& o : impl_->overflow)
    if (o) n += o->kernel_launches();
  return n;
}

void GpuEnsemble::set_state32(size_t ring, const uint32_t* x, const uint32_t* v, size_t n) {
  Impl& d = *impl_;
  if (ring >= d.params.size()) throw std::invalid_argument("ring index out of range");
  CKE(cudaSetDevice(d.device));
  if (d.overflow[ring]) {
    d.overflow[ring]->set_state32(x, v, n);
    return;
  }
  const SimParams& p = d.params[ring];
  if (n != p.car_count) throw std::invalid_argument("state length must equal ncars");
  if (d.tiled) {
    d.tpull();
    EnsRing& er = d.trings[ring];
    std::vector<uint8_t> v8(n);
    uint64_t s = 0;
    for (size_t i = 0; i < n; ++i) {
      if (x[i] >= er.L) throw std::invalid_argument("position out of range [0, length)");
      if (i && x[i - 1] >= x[i]) throw std::invalid_argument("positions must be strictly increasing");
      if (v[i] > p.v_max) throw std::invalid_argument("velocity above vmax");
      if (v[i] > er.vmax) throw std::invalid_argument("velocity above length-1 (B200 engine restriction)");
      v8[i] = static_cast<uint8_t>(v[i]);
      s += v[i];
    }
    CKE(cudaMemcpyAsync(d.ea.X[er.buf] + er.off, x, n * 4, cudaMemcpyHostToDevice, d.stream));
    CKE(cudaMemcpyAsync(d.ea.V[er.buf] + er.off, v8.data(), n, cudaMemcpyHostToDevice, d.stream));
    er.W = 0;
    er.k = 0;
    er.last_sumv = static_cast<uint32_t>(s);
    d.tpush();
    return;
  }
  d.pull();
  RingDesc& rd = d.desc[d.slot[ring]];
  std::vector<uint8_t> v8(n);
  for (size_t i = 0; i < n; ++i) {
    if (x[i] >= rd.L) throw std::invalid_argument("position out of range [0, length)");
    if (i && x[i - 1] >= x[i]) throw std::invalid_argument("positions must be strictly increasing");
    if (v[i] > p.v_max) throw std::invalid_argument("velocity above vmax");
    if (v[i] > rd.vmax) throw std::invalid_argument("velocity above length-1 (B200 engine restriction)");
    v8[i] = static_cast<uint8_t>(v[i]);
  }
  CKE(cudaMemcpyAsync(d.X + rd.off, x, n * 4, cudaMemcpyHostToDevice, d.stream));
  CKE(cudaMemcpyAsync(d.V + rd.off, v8.data(), n, cudaMemcpyHostToDevice, d.stream));
  rd.W = 0;
  rd.E = mulmod(rd.s0, powmod(kA, draw_exponent(rd.t, rd.n, 0)));
  uint64_t s = 0;
  for (size_t i = 0; i < n; ++i) s += v[i];
  rd.last_sumv = static_cast<uint32_t>(s);
  d.push();
}

void GpuEnsemble::set_state_all32(const uint32_t* x, const uint32_t* v, size_t total) {
  Impl& d = *impl_;
  CKE(cudaSetDevice(d.device));
  const size_t R = d.params.size();
  std::vector<size_t> start(R + 1, 0);
  for (size_t r = 0; r < R; ++r) start[r + 1] = start[r] + d.params[r].car_count;
  if (total != start[R]) throw std::invalid_argument("state length must equal the ensemble's total car count");
  if (!d.tiled) {  // shared-memory layout: ring by ring
    for (size_t r = 0; r < R; ++r)
      set_state32(r, x + start[r], v + start[r], start[r + 1] - start[r]);
    return;
  }
  d.tpull();
  cudaPointerAttributes pa{};
  const bool direct_x = cudaPointerGetAttributes(&pa, x) == cudaSuccess && pa.type == cudaMemoryTypeHost;
  cudaGetLastError();
  if (direct_x) {
    // positions: one DMA straight from the caller, scattered and checked on
    // the device; velocities: narrowed (rules 3-4) on the host, one DMA
    CKE(cudaMemcpyAsync(d.d_in_x, x, total * 4, cudaMemcpyHostToDevice, d.stream));
    std::atomic<unsigned long long> vcode{~0ull};
    const unsigned jobs = static_cast<unsigned>(std::min<size_t>(R, 4 * size_t(host_threads())));
    host_run(jobs, [&](unsigned j) {
      for (size_t r = j; r < R; r += jobs) {
        const uint64_t c = narrow_v32(v, start[r], start[r + 1], d.params[r].v_max, d.trings[r].vmax,
                                      d.h_stage_v, 1);
        unsigned long long m = vcode.load();
        while (c < m && !vcode.compare_exchange_weak(m, c)) {
        }
      }
    });
    const unsigned long long hc = vcode.load();
    CKE(cudaMemcpyAsync(d.d_in_v, d.h_stage_v, total, cudaMemcpyHostToDevice, d.stream));
    CKE(cudaMemsetAsync(d.d_code, 0xff, sizeof(unsigned long long), d.stream));
    ens_load_kernel<<<static_cast<unsigned>(R), 256, 0, d.stream>>>(d.ea, d.d_start, d.d_in_x, d.d_in_v, d.d_sums,
                                                                     d.d_code);
    ens_commit_kernel<<<static_cast<unsigned>((R + 255) / 256), 256, 0, d.stream>>>(d.ea, d.d_sums, d.d_code, hc);
    CKE(cudaGetLastError());
    d.launches += 2;
    CKE(cudaMemcpyAsync(d.h_code, d.d_code, sizeof(unsigned long long), cudaMemcpyDeviceToHost, d.stream));
    CKE(cudaStreamSynchronize(d.stream));
    d.dirty = true;  // the device ring records changed (committed) or not; re-read them
    const unsigned long long code = std::min<unsigned long long>(*d.h_code, hc);
    switch (code == ~0ull ? 0 : static_cast<int>(code & 3u) + 1) {
      case 1: throw std::invalid_argument("position out of range [0, length)");
      case 2: throw std::invalid_argument("positions must be strictly increasing");
      case 3: throw std::invalid_argument("velocity above vmax");
      case 4: throw std::invalid_argument("velocity above length-1 (B200 engine restriction)");
      default: break;
    }
    return;
  }
  const size_t pad = d.stage_cars;
  // rings validated and packed into the tiled layout in parallel; the
  // lowest failing ring's rule is reported
  std::vector<int> err(R, 0);
  std::vector<uint32_t> sums(R, 0);
  const unsigned jobs = static_cast<unsigned>(std::min<size_t>(R, 4 * size_t(host_threads())));
  host_run(jobs, [&](unsigned j) {
    for (size_t r = j; r < R; r += jobs) {
      const EnsRing& er = d.trings[r];
      const SimParams& p = d.params[r];
      const uint32_t* xr = x + start[r];
      const uint32_t* vr = v + start[r];
      uint32_t* ox = d.h_stage_x + er.off;
      uint8_t* ov = d.h_stage_v + er.off;
      uint64_t s = 0;
      int e = 0;
      for (size_t i = 0; i < er.n && !e; ++i) {
        if (xr[i] >= er.L) e = 1;
        else if (i && xr[i - 1] >= xr[i]) e = 2;
        else if (vr[i] > p.v_max) e = 3;
        else if (vr[i] > er.vmax) e = 4;
        ox[i] = xr[i];
        ov[i] = static_cast<uint8_t>(vr[i]);
        s += vr[i];
      }
      err[r] = e;
      sums[r] = static_cast<uint32_t>(s);
    }
  });
  for (size_t r = 0; r < R; ++r) {
    switch (err[r]) {
      case 1: throw std::invalid_argument("position out of range [0, length)");
      case 2: throw std::invalid_argument("positions must be strictly increasing");
      case 3: throw std::invalid_argument("velocity above vmax");
      case 4: throw std::invalid_argument("velocity above length-1 (B200 engine restriction)");
      default: break;
    }
  }
  // one upload into each buffer a ring reads from (the other buffer of a
  // ring is its step output, so overwriting it there is harmless)
  bool used[2] = {false, false};
  for (const EnsRing& er : d.trings) used[er.buf & 1u] = true;
  for (int b = 0; b < 2; ++b) {
    if (!used[b]) continue;
    CKE(cudaMemcpyAsync(d.ea.X[b], d.h_stage_x, pad * 4, cudaMemcpyHostToDevice, d.stream));
    CKE(cudaMemcpyAsync(d.ea.V[b], d.h_stage_v, pad, cudaMemcpyHostToDevice, d.stream));
  }
  for (size_t r = 0; r < R; ++r) {
    EnsRing& er = d.trings[r];
    er.W = 0;
    er.k = 0;
    er.last_sumv = sums[r];
  }
  d.tpush();
}

void GpuEnsemble::enqueue(uint64_t steps) {
  Impl& d = *impl_;
  CKE(cudaSetDevice(d.device));
  if (d.tiled) {
    if (steps) d.tlaunch(steps);
    return;
  }
  d.launch(steps);
  for (auto& o : d.overflow)
    if (o) o->enqueue(steps);
}

void GpuEnsemble::synchronize() {
  Impl& d = *impl_;
  CKE(cudaSetDevice(d.device));
  CKE(cudaStreamSynchronize(d.stream));
  if (d.tiled) d.tpull();  // raises on a plan contradiction
  for (auto& o : d.overflow)
    if (o) o->synchronize();
}

void GpuEnsemble::advance(uint64_t steps) {
  enqueue(steps);
  synchronize();
}

uint64_t GpuEnsemble::steps_done(size_t ring) {
  Impl& d = *impl_;
  if (ring >= d.params.size()) throw std::invalid_argument("ring index out of range");
  if (d.tiled) {
    d.tpull();
    return d.trings[ring].t;
  }
  if (d.overflow[ring]) return d.overflow[ring]->steps_done();
  d.pull();
  return d.desc[d.slot[ring]].t;
}

void GpuEnsemble::sumv_totals(uint64_t* out, size_t cap) {
  Impl& d = *impl_;
  CKE(cudaSetDevice(d.device));
  if (d.tiled) {
    d.tpull();
    for (size_t r = 0; r < d.params.size() && r < cap; ++r) out[r] = d.trings[r].sumv_total;
    return;
  }
  d.pull();
  for (size_t r = 0; r < d.params.size() && r < cap; ++r) {
    if (d.overflow[r]) {
      const size_t k = d.overflow[r]->sumv_series(nullptr, 0);
      std::vector<uint64_t> s(k);
      d.overflow[r]->sumv_series(s.data(), k);
      uint64_t tot = 0;
      for (uint64_t x : s) tot += x;
      out[r] = tot;
    } else {
      out[r] = d.desc[d.slot[r]].sumv_total;
    }
  }
}

void GpuEnsemble::sumv_last(uint64_t* out, size_t cap) {
  Impl& d = *impl_;
  CKE(cudaSetDevice(d.device));
  if (d.tiled) {
    d.tpull();
    for (size_t r = 0; r < d.params.size() && r < cap; ++r) out[r] = d.trings[r].last_sumv;
    return;
  }
  d.pull();
  for (size_t r = 0; r < d.params.size() && r < cap; ++r) {
    if (d.overflow[r]) {
      const size_t k = d.overflow[r]->sumv_series(nullptr, 0);
      std::vector<uint64_t> s(k);
      d.overflow[r]->sumv_series(s.data(), k);
      out[r] = k ? s.back() : 0;
    } else {
      out[r] = d.desc[d.slot[r]].last_sumv;
    }
  }
}

void GpuEnsemble::state(size_t ring, uint64_t* x, uint64_t* v) {
  Impl& d = *impl_;
  if (ring >= d.params.size()) throw std::invalid_argument("ring index out of range");
  CKE(cudaSetDevice(d.device));
  if (d.tiled) {
    d.tpull();
    const EnsRing& er = d.trings[ring];
    std::vector<uint32_t> hx(er.n);
    std::vector<uint8_t> hv(er.n);
    CKE(cudaMemcpyAsync(hx.data(), d.ea.X[er.buf] + er.off, size_t(er.n) * 4, cudaMemcpyDeviceToHost, d.stream));
    CKE(cudaMemcpyAsync(hv.data(), d.ea.V[er.buf] + er.off, er.n, cudaMemcpyDeviceToHost, d.stream));
    CKE(cudaStreamSynchronize(d.stream));
    const uint32_t head = (er.n - er.W) % er.n;  // rank-0 car
    for (uint32_t k = 0; k < er.n; ++k) {
      uint32_t id = head + k;
      if (id >= er.n) id -= er.n;
      if (x) x[k] = hx[id];
      if (v) v[k] = hv[id];
    }
    return;
  }
  if (d.overflow[ring]) {
    d.overflow[ring]->state(x, v);
    return;
  }
  d.pull();
  const RingDesc& rd = d.desc[d.slot[ring]];
  std::vector<uint32_t> hx(rd.n);
  std::vector<uint8_t> hv(rd.n);
  CKE(cudaMemcpyAsync(hx.data(), d.X + rd.off, size_t(rd.n) * 4, cudaMemcpyDeviceToHost, d.stream));
  CKE(cudaMemcpyAsync(hv.data(), d.V + rd.off, rd.n, cudaMemcpyDeviceToHost, d.stream));
  CKE(cudaStreamSynchronize(d.stream));
  const uint32_t head = (rd.n - rd.W) % rd.n;  // rank-0 car
  for (uint32_t k = 0; k < rd.n; ++k) {
    uint32_t id = head + k;
    if (id >= rd.n) id -= rd.n;
    if (x) x[k] = hx[id];
    if (v) v[k] = hv[id];
  }
}

}  // namespace nb200
