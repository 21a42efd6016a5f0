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
//           in shared memory from its own cars, writes them with 16-byte
//           stores (no clearing pass, no byte scatter in HBM) and counts
//           them for the next step's scan; each warp compacts its cars
//           first (lanes work on cars, not cells); per car: gap to the next
//           car of the list, the counter-based draw E_t a^rank (a^rank from
//           three 4096-entry power tables for a lane's first car, then one
//           multiply by a^32 per car); exact velocity sum and wrap count.
//           Cars landing past the block (<= vmax of them) go to a spill
//           list:
//   fixup   stores the spilled cars and adds them to their block's count.
// The count pass runs only after construction / set_state.  Steps are
// enqueued without a host round trip; the per-step records are drained in
// batches.  HBM traffic per step: about 2 L bytes.
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

// Round 2 form of the move (grid_move2_kernel + grid_fixup_kernel): each
// block moves only its OWN cars.  A car landing past the block's output
// cells (at most `look` of them per block: they start within vmax cells of
// the block's end, or wrap past L) is appended to the block's spill list
// instead, and grid_fixup_kernel stores the spilled cars after every block
// has written its cells -- no warp re-simulating the previous block's last
// cars (a serial chain of global reads the other warps waited on at the
// barrier).  The block also counts the cars it placed, so the next step's
// scan needs no separate count pass over the L cells (the fixup adds the
// spilled cars to their block's count): two passes over the cells per step
// instead of three.  Draws: Q = E a^rank once per lane, then one mulmod by
// a^32 per car.
constexpr uint32_t kSpillMax = 256;  // >= look (vmax <= 254 in the grid engine)
__global__ void __launch_bounds__(kGridTPB) grid_move2_kernel(const uint8_t* __restrict__ cells,
                                                              uint8_t* __restrict__ next,
                                                              const uint32_t* __restrict__ local,
                                                              const uint32_t* __restrict__ group,
                                                              GridArgs g, StepRec* rec, uint32_t* counts_next,
                                                              uint32_t* spill, uint32_t* spill_n) {
  constexpr uint32_t CPT = kCellsPerBlock / kGridTPB;
  constexpr int NW = kGridTPB / 32;
  __shared__ __align__(16) uint8_t s_out[kCellsPerBlock];
  __shared__ __align__(16) uint8_t s_in[kCellsPerBlock];
  __shared__ uint32_t s_w[NW];
  __shared__ uint32_t s_nspill, s_cnt;
  __shared__ uint16_t s_cx[NW][32 * CPT];  // a warp's cars: cell offset from B0, position order
  const uint32_t B0 = blockIdx.x * kCellsPerBlock;
  const uint32_t lo = B0 + threadIdx.x * CPT;
  // the block's first rank and its draw power, issued before the cells
  // load so the two global round trips overlap
  const uint32_t rank0 = __ldg(local + blockIdx.x) + __ldg(group + (blockIdx.x >> 10));
  const uint32_t Eb = mulmod_d(g.E, apow_rank(g.pw, rank0));  // E a^rank0
  reinterpret_cast<uint4*>(s_out)[threadIdx.x] = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
  if (threadIdx.x == 0) {
    s_nspill = 0;
    s_cnt = 0;
  }
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
  reinterpret_cast<uint4*>(s_in)[threadIdx.x] = make_uint4(ws[0], ws[1], ws[2], ws[3]);
  const uint32_t m16 = occ_bits4(ws[0]) | (occ_bits4(ws[1]) << 4) | (occ_bits4(ws[2]) << 8) | (occ_bits4(ws[3]) << 12);
  const uint32_t occ = __popc(m16);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = occ;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += n;
  }
  const uint32_t wcnt = __shfl_sync(0xffffffffu, incl, 31);
  if (lane == 31) s_w[warp] = incl;
  {  // compact the warp's car positions (velocities are read from s_in later)
    uint32_t m = m16, q = incl - occ;
    const uint32_t off = lo - B0;
    while (m) {
      s_cx[warp][q++] = static_cast<uint16_t>(off + __ffs(m) - 1u);
      m &= m - 1u;
    }
  }
  __syncthreads();  // also orders the s_out clear before any car lands
  uint32_t wbase = 0, nfirst = 0xffffffffu;  // cars of earlier warps; first car after this warp
  for (int w = 0; w < NW; ++w) {
    const uint32_t cw = s_w[w];
    if (w < static_cast<int>(warp)) wbase += cw;
    else if (w > static_cast<int>(warp) && cw && nfirst == 0xffffffffu) nfirst = s_cx[w][0];
  }
  const uint32_t look = min(g.vmax, g.L - 1);
  const uint32_t B1 = min(B0 + kCellsPerBlock, g.L);  // end of this block's cells
  uint32_t sum = 0, wraps = 0;
  if (lane < wcnt) {
    // the lane's first draw: E a^(rank0 + wbase + lane), wbase + lane < 4096
    uint32_t Q = mulmod_d(Eb, __ldg(g.pw + wbase + lane));
    for (uint32_t j = lane; j < wcnt; j += 32) {
      const uint32_t xo = s_cx[warp][j];
      const uint32_t x = B0 + xo;
      uint32_t gap;
      if (j + 1 < wcnt) {
        gap = min(static_cast<uint32_t>(s_cx[warp][j + 1]) - xo - 1u, look);
      } else if (nfirst != 0xffffffffu) {  // the next car is in a later warp of the block
        gap = min(nfirst - xo - 1u, look);
      } else {  // the block's last car: the cells after the block (wrapping past L)
        gap = look;
        for (uint32_t d = 1; d <= look; ++d) {
          uint32_t y = x + d;
          if (y >= g.L) y -= g.L;
          if (__ldg(cells + y) != kEmpty) {
            gap = d - 1;
            break;
          }
        }
      }
      uint32_t v = min(min(static_cast<uint32_t>(s_in[xo]) + 1, g.vmax), gap);
      const uint32_t s = Q;  // draw #(t N + rank + 1)
      Q = mulmod_d(Q, g.a32);
      if (s < g.tp && v > 0) --v;
      uint32_t nx = x + v;
      const bool wrapped = nx >= g.L;
      nx -= wrapped ? g.L : 0u;
      wraps += wrapped;
      if (nx >= B0 && nx < B1) {
        s_out[nx - B0] = static_cast<uint8_t>(v);
      } else {
        const uint32_t slot = atomicAdd(&s_nspill, 1u);
        spill[size_t(blockIdx.x) * kSpillMax + slot] = nx;
        spill[size_t(gridDim.x) * kSpillMax + size_t(blockIdx.x) * kSpillMax + slot] = v;
      }
      sum += v;
    }
  }
  __syncthreads();
  uint32_t placed = 0;
  if (B0 + (threadIdx.x + 1) * CPT <= g.L) {
    const uint4 o = reinterpret_cast<const uint4*>(s_out)[threadIdx.x];
    reinterpret_cast<uint4*>(next + B0)[threadIdx.x] = o;
    placed = (__popc(__vcmpne4(o.x, 0xffffffffu)) + __popc(__vcmpne4(o.y, 0xffffffffu)) +
              __popc(__vcmpne4(o.z, 0xffffffffu)) + __popc(__vcmpne4(o.w, 0xffffffffu))) >> 3;
  } else {
    for (uint32_t k = threadIdx.x * CPT; k < (threadIdx.x + 1) * CPT && B0 + k < g.L; ++k) {
      next[B0 + k] = s_out[k];
      placed += s_out[k] != kEmpty;
    }
  }
  sum = __reduce_add_sync(0xffffffffu, sum);
  wraps = __reduce_add_sync(0xffffffffu, wraps);
  placed = __reduce_add_sync(0xffffffffu, placed);
  if (lane == 0) {
    StepRec* r = rec + (g.t % kRecCap);
    if (sum) atomicAdd(&r->sumv, static_cast<unsigned long long>(sum));
    if (wraps) atomicAdd(&r->c, wraps);
    atomicAdd(&s_cnt, placed);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    counts_next[blockIdx.x] = s_cnt;
    spill_n[blockIdx.x] = s_nspill;
  }
}

// The spilled cars of every block into the next array (all blocks' own
// cells are written by now: stream order) and into their block's count.
__global__ void grid_fixup_kernel(const uint32_t* __restrict__ spill, const uint32_t* __restrict__ spill_n,
                                  uint32_t nb, uint8_t* next, uint32_t* counts_next) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    const uint32_t n = spill_n[b];
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t nx = spill[size_t(b) * kSpillMax + i];
      const uint32_t v = spill[size_t(nb) * kSpillMax + size_t(b) * kSpillMax + i];
      next[nx] = static_cast<uint8_t>(v);
      atomicAdd(counts_next + nx / kCellsPerBlock, 1u);
    }
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
  uint32_t* counts_next = nullptr;  // the next array's block counts (move2 + fixup)
  uint32_t *spill = nullptr, *spill_n = nullptr;
  bool counts_valid = false;  // counts[] describe cells[cur]
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
    counts_valid = true;
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
    if (!counts_valid) {  // after construction / set_state; later steps count as they move
      grid_count_kernel<<<nb, kGridTPB, 0, stream>>>(cells[cur], L, counts);
      ++launches;
    }
    scan();
    grid_move2_kernel<<<nb, kGridTPB, 0, stream>>>(cells[cur], cells[cur ^ 1], local, group, g, rec, counts_next,
                                                   spill, spill_n);
    grid_fixup_kernel<<<std::max(1u, std::min(1024u, (nb + 255) / 256)), 256, 0, stream>>>(spill, spill_n, nb,
                                                                                            cells[cur ^ 1], counts_next);
    CKG(cudaGetLastError());
    launches += 4;
    std::swap(counts, counts_next);
    counts_valid = true;
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
  CKG(cudaMalloc(&d.counts_next, size_t(d.nb) * 4));
  CKG(cudaMalloc(&d.spill, size_t(d.nb) * kSpillMax * 2 * 4));
  CKG(cudaMalloc(&d.spill_n, size_t(d.nb) * 4));
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
  cudaFree(counts_next);
  cudaFree(spill);
  cudaFree(spill_n);
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
  d.counts_valid = false;
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
