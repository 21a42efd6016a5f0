// grid.cu -- GpuGrid: the reference's cell-array engine on the GPU
// (NASCH_ENGINE_GRID_REFERENCE; src/model.cpp:77-129, src/engine.cpp:186-196).
//
// The reference keeps it as a serial equivalence oracle: cells[x] = velocity
// of the occupant or -1; each step scans the occupied cells in ascending
// order (= rank order, so draw #(t*N + rank + 1)), brakes to the distance to
// the next occupied cell, and scatters every car to (x + v) mod L.
// Here one step is four launches over L one-byte cells (0xff = empty):
//   count   occupied cells per 4096-cell block (16-byte loads, byte compares
//           in SIMD-within-a-register form)
//   scan    exclusive prefix over the block counts (rank of a block's first
//           car) in two levels: 1024 counts per block, then the group totals
//   move    block b assembles the NEXT array's cells [4096 b, 4096 b + 4096)
//           in shared memory from its own cars and the cars of the vmax
//           cells before it, and writes them with 16-byte stores (no
//           clearing pass, no byte scatter in HBM); each warp compacts its
//           cars first (lanes work on cars, not cells); per car: gap to the
//           next car of the list, the counter-based draw E_t a^rank (a^rank
//           from three 4096-entry power tables for a lane's first car, then
//           one multiply by a^32 per car); exact velocity sum and wrap count.
// Steps are enqueued without a host round trip; the per-step records are
// drained in batches.  HBM traffic per step: about 3 L bytes.
// Bit-identical to the agent engines (tests/test_gpu_grid.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine.hpp"
#include "minstd.hpp"
#include "fnv_kernels.cuh"
#include "step_kernels.cuh"

namespace nb200 {

namespace {

void check_g(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  }
}
#define CKG(call) check_g((call), #call)

constexpr uint32_t kCellsPerBlock = 4096;
constexpr int kGridTPB = 256;  // 16 cells per thread
constexpr uint8_t kEmpty = 0xff;


// Occupied bytes (!= 0xff) among the 16 cells [lo, lo + 16).
__device__ __forceinline__ uint32_t occupied16(const uint8_t* __restrict__ cells, uint32_t lo, uint32_t L) {
  if (lo + 16 <= L) {
    const uint4 w = *reinterpret_cast<const uint4*>(cells + lo);
    return (__popc(__vcmpne4(w.x, 0xffffffffu)) + __popc(__vcmpne4(w.y, 0xffffffffu)) +
            __popc(__vcmpne4(w.z, 0xffffffffu)) + __popc(__vcmpne4(w.w, 0xffffffffu))) >> 3;
  }
  uint32_t c = 0;
  for (uint32_t i = lo; i < min(L, lo + 16); ++i) c += cells[i] != kEmpty;
  return c;
}

// One thread per 16 consecutive cells of the block (as the move kernel).
__global__ void __launch_bounds__(kGridTPB) grid_count_kernel(const uint8_t* __restrict__ cells, uint32_t L,
                                                              uint32_t* counts) {
  const uint32_t b = blockIdx.x;
  const uint32_t lo = b * kCellsPerBlock + threadIdx.x * 16u;
  uint32_t c = lo < L ? occupied16(cells, lo, L) : 0u;
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ uint32_t s[kGridTPB / 32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x / 32] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kGridTPB / 32; ++w) t += s[w];
    counts[b] = t;
  }
}

// Exclusive scan of the nb block counts in two levels: grid_scan_local
// (1024 counts per block, warp-shuffle scan) writes each block's local
// prefix and the 1024-block group totals; grid_scan_top scans the <= 1024
// group totals.  A block's first rank is local[b] + top[b >> 10].
__device__ __forceinline__ uint32_t block_excl_scan_1024(uint32_t v, uint32_t* s_w, uint32_t* total) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += n;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < blockDim.x / 32 ? s_w[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t n = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= static_cast<uint32_t>(o)) wi += n;
    }
    s_w[lane] = wi - w;
    if (lane == 31) *total = wi;
  }
  __syncthreads();
  return s_w[warp] + incl - v;
}

__global__ void __launch_bounds__(1024) grid_scan_local(const uint32_t* counts, uint32_t nb, uint32_t* local,
                                                        uint32_t* group) {
  __shared__ uint32_t s_w[32], s_tot;
  const uint32_t i = blockIdx.x * 1024u + threadIdx.x;
  const uint32_t v = i < nb ? counts[i] : 0u;
  const uint32_t ex = block_excl_scan_1024(v, s_w, &s_tot);
  if (i < nb) local[i] = ex;
  if (threadIdx.x == 0) group[blockIdx.x] = s_tot;
}

__global__ void __launch_bounds__(1024) grid_scan_top(uint32_t* group, uint32_t ng) {
  __shared__ uint32_t s_w[32], s_tot;
  const uint32_t v = threadIdx.x < ng ? group[threadIdx.x] : 0u;
  const uint32_t ex = block_excl_scan_1024(v, s_w, &s_tot);
  if (threadIdx.x < ng) group[threadIdx.x] = ex;
}

struct GridArgs {
  uint32_t L, N, vmax, tp;
  uint32_t E;                 // s0 a^(t N + 1): the draw of the rank-0 car at step t
  uint32_t a32;               // a^32 (a lane's next car is 32 ranks on)
  const uint32_t* pw;         // [3][4096]: a^j, a^(4096 j), a^(4096^2 j)
  unsigned long long t;
};

// Bit k set iff byte k of w is occupied (!= 0xff), k < 4.
__device__ __forceinline__ uint32_t occ_bits4(uint32_t w) {
  return ((__vcmpne4(w, 0xffffffffu) & 0x01010101u) * 0x01020408u) >> 24;
}

// The draw of the car of rank r: E a^r, a^r from the three power tables.
__device__ __forceinline__ uint32_t apow_rank(const uint32_t* pw, uint32_t r) {
  return mulmod(mulmod(__ldg(pw + (r & 4095u)), __ldg(pw + 4096 + ((r >> 12) & 4095u))),
                __ldg(pw + 8192 + (r >> 24)));
}

// Gap ahead of the car at x by reading the cell array (any vmax, wraps).
__device__ __forceinline__ uint32_t gap_scan(const uint8_t* __restrict__ cells, uint32_t x, uint32_t look,
                                             uint32_t L) {
  for (uint32_t d = 1; d <= look; ++d) {
    uint32_t y = x + d;
    if (y >= L) y -= L;
    if (cells[y] != kEmpty) return d - 1;
  }
  return look;
}

// Block b owns the OUTPUT cells [B0, B0 + 4096) of the next array and
// assembles them in shared memory: its own cars (one thread per 16 input
// cells, as the count kernel) land there unless they pass B0 + 4096 or wrap
// past L, and the cars of the `look` cells before B0 (mod L), computed once
// more by warp 0, land there when they cross into it.  The block then
// writes its 4096 cells with 16-byte stores: no clearing pass and no
// partial-sector scatter in HBM.  Each car's velocity and crossing are
// counted by the block that owns its input cell.  Within a warp the cars of
// its 512 cells are first compacted in shared memory (position order), so
// every lane works on cars, not on empty cells, and a car's gap is the next
// entry of the list (the warp's last car reads ahead in the cell array).
__global__ void __launch_bounds__(kGridTPB) grid_move_kernel(const uint8_t* __restrict__ cells,
                                                             uint8_t* __restrict__ next,
                                                             const uint32_t* __restrict__ local,
                                                             const uint32_t* __restrict__ group,
                                                             GridArgs g, StepRec* rec) {
  constexpr uint32_t CPT = kCellsPerBlock / kGridTPB;
  static_assert(CPT == 16, "one 16-byte load per thread");
  __shared__ __align__(16) uint8_t s_out[kCellsPerBlock];
  __shared__ uint32_t s_w[kGridTPB / 32];
  __shared__ uint16_t s_cx[kGridTPB / 32][32 * CPT];  // a warp's cars: cell offset from B0 ...
  __shared__ uint8_t s_cv[kGridTPB / 32][32 * CPT];   // ... and velocity, in position order
  const uint32_t B0 = blockIdx.x * kCellsPerBlock;
  const uint32_t lo = B0 + threadIdx.x * CPT;
  reinterpret_cast<uint4*>(s_out)[threadIdx.x] = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
  uint32_t ws[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
  if (lo + CPT <= g.L) {
    const uint4 w = *reinterpret_cast<const uint4*>(cells + lo);
    ws[0] = w.x;
    ws[1] = w.y;
    ws[2] = w.z;
    ws[3] = w.w;
  } else {
#pragma unroll
    for (uint32_t k = 0; k < CPT; ++k)
      if (lo + k < g.L) ws[k / 4] = (ws[k / 4] & ~(0xffu << (8 * (k % 4)))) | (uint32_t(cells[lo + k]) << (8 * (k % 4)));
  }
  const uint32_t m16 = occ_bits4(ws[0]) | (occ_bits4(ws[1]) << 4) | (occ_bits4(ws[2]) << 8) | (occ_bits4(ws[3]) << 12);
  const uint32_t occ = __popc(m16);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // Compact the warp's cars (512 cells) into shared memory in position
  // order, then give lane l the cars l, l + 32, ...: every lane busy, the
  // gap of all but the warp's last car is the next car in the list.
  uint32_t incl = occ;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += n;
  }
  const uint32_t wcnt = __shfl_sync(0xffffffffu, incl, 31);
  if (lane == 31) s_w[warp] = incl;
  {
    uint32_t m = m16, q = incl - occ;
    while (m) {
      const uint32_t k = __ffs(m) - 1u;
      m &= m - 1u;
      s_cx[warp][q] = static_cast<uint16_t>(lo - B0 + k);
      const uint32_t wk = k < 8 ? (k < 4 ? ws[0] : ws[1]) : (k < 12 ? ws[2] : ws[3]);  // no local array
      s_cv[warp][q] = static_cast<uint8_t>(wk >> (8 * (k % 4)));
      ++q;
    }
  }
  __syncthreads();  // also orders the s_out clear before any car lands
  uint32_t wbase = 0;
  for (uint32_t w = 0; w < warp; ++w) wbase += s_w[w];
  const uint32_t rank0 = __ldg(local + blockIdx.x) + __ldg(group + (blockIdx.x >> 10));
  const uint32_t look = min(g.vmax, g.L - 1);
  const uint32_t B1 = min(B0 + kCellsPerBlock, g.L);  // end of this block's output cells
  uint32_t sum = 0, wraps = 0;
  if (lane < wcnt) {
    uint32_t ap = apow_rank(g.pw, rank0 + wbase + lane);
    for (uint32_t j = lane; j < wcnt; j += 32) {
      const uint32_t x = B0 + s_cx[warp][j];
      const uint32_t ck = s_cv[warp][j];
      const uint32_t gap = j + 1 < wcnt ? min(static_cast<uint32_t>(s_cx[warp][j + 1]) + B0 - x - 1u, look)
                                        : gap_scan(cells, x, look, g.L);
      uint32_t v = min(min(ck + 1, g.vmax), gap);
      const uint32_t s = mulmod(g.E, ap);  // draw #(t N + rank + 1)
      ap = mulmod(ap, g.a32);
      if (s < g.tp && v > 0) --v;
      uint32_t nx = x + v;
      if (nx >= g.L) {
        nx -= g.L;
        ++wraps;
      }
      if (nx >= B0 && nx < B1) s_out[nx - B0] = static_cast<uint8_t>(v);
      sum += v;
    }
  }
  // Warp 0: cars of the `look` cells before B0 (mod L) that land in this
  // block.  Their ranks count back from the block's first rank (mod N).
  if (warp == 0 && g.L > kCellsPerBlock) {
    uint32_t after = 0;  // occupied cells between the current chunk and B0
    for (uint32_t c0 = 0; c0 < look; c0 += 32) {
      const uint32_t j = c0 + lane + 1;  // cell B0 - j
      const uint32_t y = j <= look ? (B0 >= j ? B0 - j : B0 + g.L - j) : 0u;
      const bool occd = j <= look && cells[y] != kEmpty;
      const uint32_t bal = __ballot_sync(0xffffffffu, occd);
      if (occd) {
        // ranks: cars at B0-1, B0-2, ... are rank0-1, rank0-2, ...
        const uint32_t nearer = __popc(bal & ((1u << lane) - 1u));  // occupied cells closer to B0
        uint32_t r = rank0 + g.N - (after + nearer + 1);
        if (r >= g.N) r -= g.N;
        const uint32_t cy = cells[y];
        uint32_t v = min(min(cy + 1, g.vmax), gap_scan(cells, y, look, g.L));
        const uint32_t sd = mulmod(g.E, apow_rank(g.pw, r));
        if (sd < g.tp && v > 0) --v;
        uint32_t nx = y + v;
        if (nx >= g.L) nx -= g.L;
        if (nx >= B0 && nx < B1) s_out[nx - B0] = static_cast<uint8_t>(v);
      }
      after += __popc(bal);
    }
  }
  __syncthreads();
  if (B0 + (threadIdx.x + 1) * CPT <= g.L) {
    reinterpret_cast<uint4*>(next + B0)[threadIdx.x] = reinterpret_cast<const uint4*>(s_out)[threadIdx.x];
  } else {
    for (uint32_t k = threadIdx.x * CPT; k < (threadIdx.x + 1) * CPT && B0 + k < g.L; ++k) next[B0 + k] = s_out[k];
  }
  sum = __reduce_add_sync(0xffffffffu, sum);
  wraps = __reduce_add_sync(0xffffffffu, wraps);
  if (lane == 0) {
    StepRec* r = rec + (g.t % kRecCap);
    if (sum) atomicAdd(&r->sumv, static_cast<unsigned long long>(sum));
    if (wraps) atomicAdd(&r->c, wraps);
  }
}

__global__ void grid_compact_kernel(const uint8_t* __restrict__ cells, uint32_t L,
                                    const uint32_t* __restrict__ local, const uint32_t* __restrict__ group,
                                    uint32_t* xs, uint8_t* vs) {
  constexpr uint32_t CPT = kCellsPerBlock / kGridTPB;
  const uint32_t lo = blockIdx.x * kCellsPerBlock + threadIdx.x * CPT;
  uint32_t occ = 0;
  for (uint32_t k = 0; k < CPT; ++k) occ += (lo + k < L) && cells[lo + k] != kEmpty;
  uint32_t incl = occ;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += n;
  }
  __shared__ uint32_t s_w[kGridTPB / 32];
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  uint32_t r = local[blockIdx.x] + group[blockIdx.x >> 10] + incl - occ;
  for (uint32_t w = 0; w < warp; ++w) r += s_w[w];
  for (uint32_t k = 0; k < CPT; ++k) {
    if (lo + k < L && cells[lo + k] != kEmpty) {
      xs[r] = lo + k;
      vs[r] = cells[lo + k];
      ++r;
    }
  }
}

__global__ void grid_init_kernel(uint8_t* cells, uint32_t L, uint32_t N) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x)
    cells[i * L / N] = 0;  // model.cpp:30-40 then agent_to_grid, model.cpp:77-85
}

}  // namespace

struct GpuGrid::Impl {
  SimParams params;
  int device = 0;
  cudaStream_t stream = nullptr;
  uint32_t L = 0, N = 0, vmax = 0, nb = 0;
  uint8_t* cells[2] = {nullptr, nullptr};
  int cur = 0;
  uint32_t *counts = nullptr, *local = nullptr, *group = nullptr, *xs = nullptr;
  uint32_t ng = 0;  // 1024-block groups of the two-level scan
  uint8_t* vs = nullptr;
  StepRec* rec = nullptr;
  StepRec* hrec = nullptr;  // pinned [kRecCap]
  uint32_t* pw = nullptr;   // device power tables (GridArgs::pw)
  uint64_t drained = 0;
  uint32_t* hx = nullptr;
  uint8_t* hv = nullptr;
  uint64_t steps_done = 0, hash = kFnvBasis, launches = 0, sumv0 = 0;
  bool checksum_on = true;
  std::vector<uint64_t> sumv_host, wraps_host;
  std::vector<Frame> frames;
  // on-device checksum (fnv_kernels.cuh): chunk maps of the compacted,
  // rank-ordered row, composed and applied to a device digest
  unsigned long long* fT[2] = {nullptr, nullptr};
  unsigned long long* fP[2] = {nullptr, nullptr};
  unsigned long long* dhash = nullptr;
  ~Impl();

  void scan() {
    grid_scan_local<<<ng, 1024, 0, stream>>>(counts, nb, local, group);
    grid_scan_top<<<1, 1024, 0, stream>>>(group, ng);
  }

  void compact() {
    grid_count_kernel<<<nb, kGridTPB, 0, stream>>>(cells[cur], L, counts);
    scan();
    grid_compact_kernel<<<nb, kGridTPB, 0, stream>>>(cells[cur], L, local, group, xs, vs);
    CKG(cudaGetLastError());
    launches += 4;
  }

  // Folds the current row (positions, then velocities) into the device
  // digest: no transfer of the state.
  void hash_step() {
    const uint32_t nch = (N + kFnvChunk - 1) / kFnvChunk;
    if (!dhash) {
      for (int b = 0; b < 2; ++b) {
        CKG(cudaMalloc(&fT[b], size_t(2) * nch * 256 * sizeof(unsigned long long)));
        CKG(cudaMalloc(&fP[b], size_t(2) * nch * sizeof(unsigned long long)));
      }
      CKG(cudaMalloc(&dhash, sizeof(unsigned long long)));
      CKG(cudaMemcpyAsync(dhash, &hash, sizeof hash, cudaMemcpyHostToDevice, stream));
    }
    compact();
    fnv_slice_chunk_kernel<uint32_t><<<nch, 256, 0, stream>>>(xs, N, fT[0], fP[0]);
    fnv_slice_chunk_kernel<uint8_t><<<nch, 256, 0, stream>>>(vs, N, fT[0] + size_t(nch) * 256, fP[0] + nch);
    int in = 0;
    for (uint32_t m = 2 * nch; m > 1; m = (m + 1) / 2) {
      fnv_compose_kernel<<<(m + 1) / 2, 256, 0, stream>>>(fT[in], fP[in], m, fT[in ^ 1], fP[in ^ 1]);
      in ^= 1;
    }
    fnv_apply_kernel<<<1, 1, 0, stream>>>(fT[in], fP[in], dhash);
    CKG(cudaGetLastError());
    launches += 4;
  }

  void pull_hash() {
    if (!dhash) return;
    CKG(cudaMemcpyAsync(&hash, dhash, sizeof hash, cudaMemcpyDeviceToHost, stream));
    CKG(cudaStreamSynchronize(stream));
  }

  // One step, enqueued: no host round trip (records drained in batches).
  void step() {
    if (steps_done - drained >= kRecCap / 2) drain();
    const uint32_t E = mulmod(seeded(params.seed), powmod(kA, draw_exponent(steps_done, N, 0)));
    const GridArgs g{L, N, vmax, deceleration_threshold(params.p), E, powmod(kA, 32), pw, steps_done};
    CKG(cudaMemsetAsync(rec + (steps_done % kRecCap), 0, sizeof(StepRec), stream));
    grid_count_kernel<<<nb, kGridTPB, 0, stream>>>(cells[cur], L, counts);
    scan();
    grid_move_kernel<<<nb, kGridTPB, 0, stream>>>(cells[cur], cells[cur ^ 1], local, group, g, rec);
    CKG(cudaGetLastError());
    launches += 4;
    cur ^= 1;
    ++steps_done;
  }

  // Per-step records of [drained, steps_done) to the host series.
  void drain() {
    if (drained == steps_done) return;
    const uint64_t first = drained, count = steps_done - drained;
    uint64_t done = 0;
    while (done < count) {
      const uint64_t slot = (first + done) % kRecCap;
      const uint64_t seg = std::min<uint64_t>(count - done, kRecCap - slot);
      CKG(cudaMemcpyAsync(hrec + done, rec + slot, seg * sizeof(StepRec), cudaMemcpyDeviceToHost, stream));
      done += seg;
    }
    CKG(cudaStreamSynchronize(stream));
    for (uint64_t k = 0; k < count; ++k) {
      sumv_host.push_back(hrec[k].sumv);
      wraps_host.push_back(hrec[k].c);
    }
    drained = steps_done;
  }

  // grid_to_agent (model.cpp:87-97): occupied cells in ascending order.
  void fetch() {
    compact();
    CKG(cudaMemcpyAsync(hx, xs, size_t(N) * 4, cudaMemcpyDeviceToHost, stream));
    CKG(cudaMemcpyAsync(hv, vs, N, cudaMemcpyDeviceToHost, stream));
    CKG(cudaStreamSynchronize(stream));
  }

  bool frame_due() const {
    return params.output_mode != OutputMode::none && steps_done < params.steps &&
           steps_done % params.output_stride == 0;
  }

  void record_frame() {
    Frame f;
    f.step = steps_done;
    f.positions.assign(hx, hx + N);
    f.velocities.assign(hv, hv + N);
    frames.push_back(std::move(f));
  }
};

GpuGrid::GpuGrid(const SimParams& p) : impl_(new Impl) {
  Impl& d = *impl_;
  p.validate();
  d.params = p;
  if (p.road_length > 0xffffffffull - kCellsPerBlock)
    throw std::invalid_argument("length too large for the grid engine");
  if (std::min<uint64_t>(p.v_max, p.road_length - 1) > 254)
    throw std::invalid_argument("the grid engine stores velocities in one byte (vmax <= 254)");
  int ndev = 0;
  const cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    throw std::runtime_error(std::string("no CUDA device available for the B200 engine (") +
                             cudaGetErrorString(e) + ")");
  CKG(cudaGetDevice(&d.device));
  d.L = static_cast<uint32_t>(p.road_length);
  d.N = static_cast<uint32_t>(p.car_count);
  d.vmax = static_cast<uint32_t>(std::min<uint64_t>(p.v_max, p.road_length - 1));
  d.nb = (d.L + kCellsPerBlock - 1) / kCellsPerBlock;
  CKG(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
  for (int b = 0; b < 2; ++b) CKG(cudaMalloc(&d.cells[b], d.L));
  CKG(cudaMalloc(&d.counts, size_t(d.nb) * 4));
  d.ng = (d.nb + 1023) / 1024;
  CKG(cudaMalloc(&d.local, size_t(d.nb) * 4));
  CKG(cudaMalloc(&d.group, size_t(d.ng) * 4));
  CKG(cudaMalloc(&d.xs, size_t(d.N) * 4));
  CKG(cudaMalloc(&d.vs, d.N));
  CKG(cudaMalloc(&d.rec, sizeof(StepRec) * kRecCap));
  CKG(cudaMallocHost(&d.hrec, sizeof(StepRec) * kRecCap));
  {
    std::vector<uint32_t> tab(3 * 4096);
    for (int k = 0; k < 3; ++k) {
      const uint32_t step = powmod(kA, uint64_t(1) << (12 * k));
      tab[k * 4096] = 1;
      for (int j = 1; j < 4096; ++j) tab[k * 4096 + j] = mulmod(tab[k * 4096 + j - 1], step);
    }
    CKG(cudaMalloc(&d.pw, tab.size() * 4));
    CKG(cudaMemcpy(d.pw, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice));
  }
  CKG(cudaMallocHost(&d.hx, size_t(d.N) * 4));
  CKG(cudaMallocHost(&d.hv, d.N));
  CKG(cudaMemsetAsync(d.cells[0], kEmpty, d.L, d.stream));
  grid_init_kernel<<<std::max(1u, std::min(4096u, (d.N + 255) / 256)), 256, 0, d.stream>>>(d.cells[0], d.L, d.N);
  CKG(cudaGetLastError());
  CKG(cudaStreamSynchronize(d.stream));
  if (d.frame_due()) {
    d.fetch();
    d.record_frame();
  }
}

// Released by Impl's destructor: nothing leaks if construction throws.
GpuGrid::Impl::~Impl() {
  cudaSetDevice(device);
  if (stream) cudaStreamSynchronize(stream);
  for (int b = 0; b < 2; ++b) cudaFree(cells[b]);
  cudaFree(counts);
  cudaFree(local);
  cudaFree(group);
  cudaFree(xs);
  cudaFree(vs);
  cudaFree(rec);
  cudaFree(pw);
  for (int b = 0; b < 2; ++b) {
    cudaFree(fT[b]);
    cudaFree(fP[b]);
  }
  cudaFree(dhash);
  cudaFreeHost(hrec);
  cudaFreeHost(hx);
  cudaFreeHost(hv);
  if (stream) cudaStreamDestroy(stream);
}

GpuGrid::~GpuGrid() = default;

void GpuGrid::set_state(const uint64_t* x, const uint64_t* v, size_t n) {
  Impl& d = *impl_;
  if (n != d.N) throw std::invalid_argument("state length must equal ncars");
  d.drain();
  std::vector<uint8_t> cells(d.L, kEmpty);
  uint64_t s = 0;
  for (size_t i = 0; i < n; ++i) {
    if (x[i] >= d.L) throw std::invalid_argument("position out of range [0, length)");
    if (i && x[i - 1] >= x[i]) throw std::invalid_argument("positions must be strictly increasing");
    if (v[i] > d.params.v_max) throw std::invalid_argument("velocity above vmax");
    if (v[i] > 254) throw std::invalid_argument("velocity above 254 (grid engine restriction)");
    cells[x[i]] = static_cast<uint8_t>(v[i]);
    s += v[i];
  }
  CKG(cudaMemcpyAsync(d.cells[d.cur], cells.data(), d.L, cudaMemcpyHostToDevice, d.stream));
  CKG(cudaStreamSynchronize(d.stream));
  d.sumv0 = s;
  d.sumv_host.clear();
  d.wraps_host.clear();
  if (d.steps_done == 0) {
    d.frames.clear();
    if (d.frame_due()) {
      d.fetch();
      d.record_frame();
    }
  }
}

void GpuGrid::set_state32(const uint32_t* x, const uint32_t* v, size_t n) {
  std::vector<uint64_t> x64(x, x + n), v64(v, v + n);
  set_state(x64.data(), v64.data(), n);
}

void GpuGrid::advance(uint64_t steps) {
  Impl& d = *impl_;
  CKG(cudaSetDevice(d.device));
  const uint64_t count = std::min(steps, d.params.steps - d.steps_done);
  for (uint64_t k = 0; k < count; ++k) {  // engine.cpp:186-196
    d.step();
    if (d.checksum_on) d.hash_step();
    if (d.frame_due()) {
      d.fetch();
      d.record_frame();
    }
  }
  d.drain();
}

// Asynchronous form: the steps are enqueued; synchronize() completes them.
void GpuGrid::enqueue(uint64_t steps) {
  Impl& d = *impl_;
  CKG(cudaSetDevice(d.device));
  if (d.checksum_on || d.params.output_mode != OutputMode::none) {
    advance(steps);
    return;
  }
  const uint64_t count = std::min(steps, d.params.steps - d.steps_done);
  for (uint64_t k = 0; k < count; ++k) d.step();
}
void GpuGrid::synchronize() {
  CKG(cudaSetDevice(impl_->device));
  impl_->drain();
  CKG(cudaStreamSynchronize(impl_->stream));
}
uint64_t GpuGrid::steps_done() const { return impl_->steps_done; }
uint64_t GpuGrid::checksum() const {
  CKG(cudaSetDevice(impl_->device));
  impl_->pull_hash();
  return impl_->hash;
}
const std::vector<Frame>& GpuGrid::frames() const { return impl_->frames; }
const SimParams& GpuGrid::params() const { return impl_->params; }

void GpuGrid::observables(double* density, double* mean_velocity, double* flow) {
  Impl& d = *impl_;
  CKG(cudaSetDevice(d.device));
  d.drain();
  const uint64_t total = d.sumv_host.empty() ? d.sumv0 : d.sumv_host.back();
  const double n = static_cast<double>(d.params.car_count);
  const double mean = static_cast<double>(total) / n;
  const double dens = n / static_cast<double>(d.params.road_length);
  if (density) *density = dens;
  if (mean_velocity) *mean_velocity = mean;
  if (flow) *flow = dens * mean;
}

void GpuGrid::state(uint64_t* positions, uint64_t* velocities) {
  Impl& d = *impl_;
  CKG(cudaSetDevice(d.device));
  d.fetch();
  for (uint32_t i = 0; i < d.N; ++i) {
    if (positions) positions[i] = d.hx[i];
    if (velocities) velocities[i] = d.hv[i];
  }
}

size_t GpuGrid::sumv_series(uint64_t* out, size_t cap) {
  Impl& d = *impl_;
  CKG(cudaSetDevice(d.device));
  d.drain();
  const size_t k = std::min(cap, d.sumv_host.size());
  if (out) std::memcpy(out, d.sumv_host.data(), k * sizeof(uint64_t));
  return d.sumv_host.size();
}

size_t GpuGrid::wrap_series(uint64_t* out, size_t cap) {
  Impl& d = *impl_;
  CKG(cudaSetDevice(d.device));
  d.drain();
  const size_t k = std::min(cap, d.wraps_host.size());
  if (out) std::memcpy(out, d.wraps_host.data(), k * sizeof(uint64_t));
  return d.wraps_host.size();
}

void GpuGrid::set_checksum(bool enabled) { impl_->checksum_on = enabled; }
void* GpuGrid::cuda_stream() const { return impl_->stream; }
uint64_t GpuGrid::kernel_launches() const { return impl_->launches; }
int GpuGrid::steps_per_launch() const { return 1; }
void GpuGrid::shard_range(uint64_t* first, uint64_t* count) const {
  if (first) *first = 0;
  if (count) *count = impl_->N;
}

}  // namespace nb200
