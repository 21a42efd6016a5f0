// grid.cu -- GpuGrid: the reference's cell-array engine on the GPU
// (NASCH_ENGINE_GRID_REFERENCE; src/model.cpp:77-129, src/engine.cpp:186-196).
//
// The reference keeps it as a serial equivalence oracle: cells[x] = velocity
// of the occupant or -1; each step scans the occupied cells in ascending
// order (= rank order, so draw #(t*N + rank + 1)), brakes to the distance to
// the next occupied cell, and scatters every car to (x + v) mod L.
// Here one step is four launches over L one-byte cells (0xff = empty), in
// 8192-cell blocks:
//   fixup   the previous move's spilled cars into the array and their
//           blocks' counts
//   scan    exclusive prefix over the block counts (rank of each block's
//           first car, and a^rank for its draws) in two levels; this step's
//           record zeroed
//   move    block b assembles the NEXT array's cells [8192 b, 8192 b + 8192)
//           in shared memory from its own cars, writes them with 16-byte
//           stores (no clearing pass, no byte scatter in HBM) and counts
//           them for the next step's scan; the block compacts its cars into
//           one list first (threads work on cars, not cells), with the first
//           car after the block as a sentinel; per car: gap to the next list
//           entry, the counter-based draw E_t a^rank (one multiply by
//           a^256 per car), exact velocity sum and wrap count.  Cars landing
//           past the block (<= vmax of them) go to a spill list, stored by
//           the next step's fixup (or before a state read).
// A count pass runs only after construction / set_state.  Steps are
// enqueued without a host round trip; the per-step records are drained in
// batches.  HBM traffic per step: about 2 L bytes.
// Bit-identical to the agent engines (tests/test_gpu_grid.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine.hpp"
#include "minstd.hpp"
#include "fnv_pipeline.cuh"
#include "grid_bits.cuh"
#include "step_kernels.cuh"

namespace nb200 {

namespace {

void check_g(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  }
}
#define CKG(call) check_g((call), #call)

constexpr uint32_t kCellsPerBlock = 8192;
constexpr int kGridTPB = 256;  // 32 cells per thread
constexpr uint8_t kEmpty = 0xff;
constexpr uint32_t kSpillMax = 256;  // spilled cars per block: >= look (vmax <= 254 in the grid engine)


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

// One thread per 32 consecutive cells of the block (as the move kernel).
__global__ void __launch_bounds__(kGridTPB) grid_count_kernel(const uint8_t* __restrict__ cells, uint32_t L,
                                                              uint32_t* counts) {
  const uint32_t b = blockIdx.x;
  const uint32_t lo = b * kCellsPerBlock + threadIdx.x * 32u;
  uint32_t c = (lo < L ? occupied16(cells, lo, L) : 0u) + (lo + 16 < L ? occupied16(cells, lo + 16, L) : 0u);
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

// Exclusive scan of 1024 values over one block (warp-shuffle scans).
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

// The draw of the car of rank r: E a^r, a^r from the three power tables
// pw = [a^j, a^(4096 j), a^(4096^2 j)], j < 4096.
__device__ __forceinline__ uint32_t apow_rank(const uint32_t* pw, uint32_t r) {
  return mulmod(mulmod(__ldg(pw + (r & 4095u)), __ldg(pw + 4096 + ((r >> 12) & 4095u))),
                __ldg(pw + 8192 + (r >> 24)));
}

// The exclusive scan of the block counts in two levels: grid_scan_local
// (1024 counts per block) writes each block's local prefix and a^prefix and
// the 1024-block group totals; grid_scan_top scans the group totals (and
// their a^prefix) and zeroes this step's record.  A block's first rank is
// local[b] + group[b >> 10]; its draw power plocal[b] * pgroup[b >> 10]
// reaches the move kernel as two independent loads (round 2: a rank load
// then three dependent table loads).  (A single-block scan fused with the
// spill fixup measured 23 us against ~10 us for these two launches.)
__global__ void __launch_bounds__(1024) grid_scan_local(const uint32_t* counts, uint32_t nb, uint32_t* local,
                                                        uint32_t* group, const uint32_t* pw, uint32_t* plocal) {
  __shared__ uint32_t s_w[32], s_tot;
  const uint32_t i = blockIdx.x * 1024u + threadIdx.x;
  const uint32_t v = i < nb ? counts[i] : 0u;
  const uint32_t ex = block_excl_scan_1024(v, s_w, &s_tot);
  if (i < nb) {
    local[i] = ex;
    plocal[i] = apow_rank(pw, ex);
  }
  if (threadIdx.x == 0) group[blockIdx.x] = s_tot;
}

__global__ void __launch_bounds__(1024) grid_scan_top(uint32_t* group, uint32_t ng, const uint32_t* pw,
                                                      uint32_t* pgroup, StepRec* zero) {
  __shared__ uint32_t s_w[32], s_tot;
  const uint32_t v = threadIdx.x < ng ? group[threadIdx.x] : 0u;
  const uint32_t ex = block_excl_scan_1024(v, s_w, &s_tot);
  if (threadIdx.x < ng) {
    group[threadIdx.x] = ex;
    pgroup[threadIdx.x] = apow_rank(pw, ex);
  }
  if (zero && threadIdx.x == 0) {
    zero->sumv = 0;
    zero->c = 0;
  }
}

struct GridArgs {
  uint32_t L, N, vmax, tp;
  uint32_t E;                 // s0 a^(t N + 1): the draw of the rank-0 car at step t
  uint32_t astep2;            // 2 a^kGridTPB (a thread's next car is kGridTPB ranks on; doubled: mulmod_x2)
  const uint32_t* pw;         // [3][4096]: a^j, a^(4096 j), a^(4096^2 j)
  unsigned long long t;
};

// Bit k set iff byte k of w is occupied (!= 0xff), k < 4.
__device__ __forceinline__ uint32_t occ_bits4(uint32_t w) {
  return ((__vcmpne4(w, 0xffffffffu) & 0x01010101u) * 0x01020408u) >> 24;
}

// Occupied cells of a 4-cell word as 4 bits; with velocities below 128 an
// occupied byte is one with bit 7 clear (empty = 0xff): ~w & 0x80808080,
// the four flags gathered by one multiply (bits 7+8k -> 21+k, no carries).
template <bool SMALLV>
__device__ __forceinline__ uint32_t occ4(uint32_t w) {
  if constexpr (SMALLV) {
    return ((~w & 0x80808080u) * 0x204081u) >> 28;  // bits 7, 15, 23, 31 -> 28..31
  } else {
    return occ_bits4(w);
  }
}

// Offset from B1 of the first occupied cell at or after B1 (cyclic, read
// from the current array), searched over max(16, look) cells; the window
// size when there is none (the gap is then capped at look anyway).
__device__ __forceinline__ uint32_t grid_next_car(const uint8_t* __restrict__ cells, uint32_t B1, uint32_t L,
                                                  uint32_t look) {
  const uint32_t n0 = B1 == L ? 0u : B1;  // B1 is a multiple of the block size, or L
  if (n0 + 16 <= L) {
    const uint4 w = *reinterpret_cast<const uint4*>(cells + n0);
    const uint32_t m = occ_bits4(w.x) | (occ_bits4(w.y) << 4) | (occ_bits4(w.z) << 8) | (occ_bits4(w.w) << 12);
    if (m) return __ffs(m) - 1u;
    if (look <= 16) return 16;
    for (uint32_t d = 16; d < look; ++d)
      if (cells[(n0 + d) % L] != kEmpty) return d;
    return look;
  }
  const uint32_t win = max(16u, look);
  for (uint32_t d = 0; d < win; ++d)
    if (cells[(n0 + d) % L] != kEmpty) return d;
  return win;
}

// The move (grid_move3_kernel + grid_fixup_kernel): each block moves only its
// OWN cars.  A car landing past the block's output cells (at most `look` of
// them per block: they start within vmax cells of the block's end, or wrap
// past L) is appended to the block's spill list instead, and
// grid_fixup_kernel stores the spilled cars after every block has written
// its cells.  The block also counts the cars it placed, so the next step's
// scan needs no count pass over the L cells.  Round 3 form: 8192 cells per
// block (32 per thread) to halve the per-cell share of the block's fixed
// work; the cars compacted into ONE block-wide list (offsets from B0) with a
// sentinel after the last car (the first car at or after B1, loaded with the
// block's cells), so every car's gap is list[j+1] - list[j] - 1 with no warp
// or block boundary case; thread t takes cars t, t + 256, ... (block-local
// rank j: draw E a^(rank0 + j) = Eb a^j, one mulmod by a^256 per car).
template <bool SMALLV>
__global__ void __launch_bounds__(kGridTPB) grid_move3_kernel(const uint8_t* __restrict__ cells,
                                                              uint8_t* __restrict__ next,
                                                              const uint32_t* __restrict__ plocal,
                                                              const uint32_t* __restrict__ pgroup,
                                                              GridArgs g, StepRec* rec, uint32_t* counts_next,
                                                              uint32_t* spill, uint32_t* spill_n) {
  constexpr uint32_t CPT = kCellsPerBlock / kGridTPB;  // 32
  constexpr int NW = kGridTPB / 32;
  __shared__ __align__(16) uint8_t s_out[kCellsPerBlock];
  __shared__ __align__(16) uint8_t s_in[kCellsPerBlock];
  __shared__ uint16_t s_list[kCellsPerBlock + 1];  // the block's cars (offsets from B0), then the sentinel
  __shared__ uint32_t s_w[NW];
  __shared__ uint32_t s_nspill;
  const uint32_t B0 = blockIdx.x * kCellsPerBlock;
  const uint32_t lo = B0 + threadIdx.x * CPT;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t look = min(g.vmax, g.L - 1);
  const uint32_t B1 = min(B0 + kCellsPerBlock, g.L);  // end of this block's cells
  // every global load first: the cells, the block's draw powers, a^tid
  uint32_t ws[8];
  if (lo + CPT <= g.L) {
    const uint4 u0 = *reinterpret_cast<const uint4*>(cells + lo);
    const uint4 u1 = *reinterpret_cast<const uint4*>(cells + lo + 16);
    ws[0] = u0.x; ws[1] = u0.y; ws[2] = u0.z; ws[3] = u0.w;
    ws[4] = u1.x; ws[5] = u1.y; ws[6] = u1.z; ws[7] = u1.w;
  } else {
#pragma unroll
    for (uint32_t k = 0; k < 8; ++k) ws[k] = 0xffffffffu;
    for (uint32_t k = 0; k < CPT && lo + k < g.L; ++k) {
      const uint32_t sh = 8 * (k % 4);
#pragma unroll
      for (uint32_t q = 0; q < 8; ++q)
        if (q == k / 4) ws[q] = (ws[q] & ~(0xffu << sh)) | (uint32_t(cells[lo + k]) << sh);
    }
  }
  const uint32_t pl = __ldg(plocal + blockIdx.x), pg = __ldg(pgroup + (blockIdx.x >> 10));
  const uint32_t at = __ldg(g.pw + threadIdx.x);  // a^tid
  uint32_t sentinel = 0;
  if (threadIdx.x == 0) {
    s_nspill = 0;
    sentinel = (B1 - B0) + grid_next_car(cells, B1, g.L, look);
  }
  uint4* so = reinterpret_cast<uint4*>(s_out);
  so[2 * threadIdx.x] = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
  so[2 * threadIdx.x + 1] = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
  uint4* si = reinterpret_cast<uint4*>(s_in);
  si[2 * threadIdx.x] = make_uint4(ws[0], ws[1], ws[2], ws[3]);
  si[2 * threadIdx.x + 1] = make_uint4(ws[4], ws[5], ws[6], ws[7]);
  uint32_t m = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) m |= occ4<SMALLV>(ws[q]) << (4 * q);
  const uint32_t occ = __popc(m);
  uint32_t incl = occ;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += n;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  const uint32_t cw = lane < static_cast<uint32_t>(NW) ? s_w[lane] : 0u;
  const uint32_t wbase = __reduce_add_sync(0xffffffffu, lane < warp ? cw : 0u);
  const uint32_t ncars = __reduce_add_sync(0xffffffffu, cw);
  {  // compaction into the block-wide list
    uint32_t q = wbase + incl - occ;
    const uint32_t off = lo - B0;
    while (m) {
      s_list[q++] = static_cast<uint16_t>(off + __ffs(m) - 1u);
      m &= m - 1u;
    }
  }
  if (threadIdx.x == 0) s_list[ncars] = static_cast<uint16_t>(sentinel);
  __syncthreads();  // also orders the s_out clear before any car lands
  const uint32_t Eb = mulmod_d(mulmod_d(g.E, pl), pg);  // E a^rank0
  uint32_t Q = mulmod_d(Eb, at);                        // draw of block-local car tid
  uint32_t sum = 0, wraps = 0;
  for (uint32_t j = threadIdx.x; j < ncars; j += kGridTPB) {
    const uint32_t xo = s_list[j];
    const uint32_t gap = min(static_cast<uint32_t>(s_list[j + 1]) - xo - 1u, look);
    uint32_t v = min(min(static_cast<uint32_t>(s_in[xo]) + 1, g.vmax), gap);
    const uint32_t s = Q;  // draw #(t N + rank + 1)
    Q = mulmod_x2(g.astep2, Q);
    if (s < g.tp && v > 0) --v;
    uint32_t nx = B0 + xo + v;
    const bool wrapped = nx >= g.L;
    nx -= wrapped ? g.L : 0u;
    wraps += wrapped;
    if (nx - B0 < B1 - B0) {
      s_out[nx - B0] = static_cast<uint8_t>(v);
    } else {
      const uint32_t slot = atomicAdd(&s_nspill, 1u);
      spill[size_t(blockIdx.x) * kSpillMax + slot] = nx;
      spill[size_t(gridDim.x) * kSpillMax + size_t(blockIdx.x) * kSpillMax + slot] = v;
    }
    sum += v;
  }
  __syncthreads();
  if (lo + CPT <= g.L) {
    reinterpret_cast<uint4*>(next + lo)[0] = so[2 * threadIdx.x];
    reinterpret_cast<uint4*>(next + lo)[1] = so[2 * threadIdx.x + 1];
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
  if (threadIdx.x == 0) {
    // the cars placed in this block's cells: all of its own but the spilled
    // ones (grid_fixup_kernel counts those into their destination block)
    counts_next[blockIdx.x] = ncars - s_nspill;
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
  uint32_t *plocal = nullptr, *pgroup = nullptr;  // a^prefix of the two scan levels
  uint32_t ng = 0;  // 1024-block groups of the two-level scan
  bool fixup_pending = false;  // the last move's spilled cars are not yet in cells[cur]
  uint32_t* counts_next = nullptr;  // the next array's block counts (move2 + fixup)
  uint32_t *spill = nullptr, *spill_n = nullptr;
  bool counts_valid = false;  // counts[] describe cells[cur]
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
  // on-device checksum: the nibble-decomposed digest (fnv_pipeline.cuh) of
  // the compacted, rank-ordered row
  FnvRowDigest digest;
  Ctl* dctl = nullptr;   // the compacted row's control block: W = 0, buf = 0
  RingArgs rowargs{};    // (xs, vs) as a RingArgs for the digest kernels
  // Bit-plane form (grid_bits.cuh; vmax <= 7 and L a multiple of 32): the
  // planes are the state the steps run on; cells[cur] only carries a loaded
  // state to the pack.  The readers (state, frames, checksum) compact their
  // rank-ordered row from the planes.
  bool bitmode = false;
  uint4* planes[2] = {nullptr, nullptr};
  uint4* carry[2] = {nullptr, nullptr};  // per block: the cars carried over its end by the last move
  uint32_t* bcounts = nullptr;  // cars per move block, for the scan after a pack
  uint32_t* prank = nullptr;  // a^(rank of each block's first car), kept current by the moves
  int pcur = 0;
  uint32_t nwords = 0, nbb = 0;
  int wpt = 2;  // words per thread of the move kernel (grid_bits.cuh)
  bool planes_valid = false;  // planes[pcur] (+ carry[pcur]) hold the current state
  bool cells_valid = true;    // cells[cur] holds the current state
  ~Impl();

  // cells[cur] -> planes (after construction / set_state).
  void pack() {
    gridbits::grid_pack_kernel<<<(nwords + 255) / 256, 256, 0, stream>>>(cells[cur], nwords, planes[pcur]);
    CKG(cudaMemsetAsync(carry[pcur], 0, size_t(nbb) * sizeof(uint4), stream));
    gridbits::grid_bitcount_kernel<<<nbb, gridbits::kTPB, 0, stream>>>(planes[pcur], nwords, wpt, bcounts);
    gridbits::grid_bits_scan_kernel<<<1, gridbits::kTPB, 0, stream>>>(bcounts, carry[pcur], nbb, pw,
                                                                     prank, rec + (steps_done % kRecCap));
    CKG(cudaGetLastError());
    launches += 3;
    planes_valid = true;
  }

  template <int VMAX, int WPT>
  void launch_bitmove_w(const gridbits::BitArgs& g) {
    gridbits::grid_bitmove_kernel<VMAX, WPT><<<nbb, gridbits::kTPB, 0, stream>>>(
        planes[pcur], planes[pcur ^ 1], carry[pcur], carry[pcur ^ 1], prank, g, rec);
  }
  template <int VMAX>
  void launch_bitmove(const gridbits::BitArgs& g) {
    if (wpt == 4) launch_bitmove_w<VMAX, 4>(g);
    else if (wpt == 2) launch_bitmove_w<VMAX, 2>(g);
    else launch_bitmove_w<VMAX, 1>(g);
  }

  void step_bits() {
    if (steps_done - drained >= kRecCap / 2) drain();
    if (!planes_valid) pack();
    const uint32_t E = mulmod(seeded(params.seed), powmod(kA, draw_exponent(steps_done, N, 0)));
    gridbits::BitArgs g{nwords, deceleration_threshold(params.p), E, 2 * kA, 1u, 2u,
                        {1u, 2u, 4u, 8u, 16u, 32u, 64u, 128u}, {}, {}, pw, steps_done};
    const uint32_t ainv1 = powmod(kA, kOrder - 1);  // a^-1 (Fermat)
    g.apw[0] = g.ainv[0] = 1;
    for (int k = 1; k < 8; ++k) {
      g.apw[k] = mulmod(g.apw[k - 1], kA);
      g.ainv[k] = mulmod(g.ainv[k - 1], ainv1);
    }
    switch (vmax) {
      case 1: launch_bitmove<1>(g); break;
      case 2: launch_bitmove<2>(g); break;
      case 3: launch_bitmove<3>(g); break;
      case 4: launch_bitmove<4>(g); break;
      case 5: launch_bitmove<5>(g); break;
      case 6: launch_bitmove<6>(g); break;
      default: launch_bitmove<7>(g); break;
    }
    CKG(cudaGetLastError());
    ++launches;
    pcur ^= 1;
    cells_valid = false;
    ++steps_done;
  }

  // The last move's spilled cars into cells[cur] and counts (when a state
  // read comes before the next step).
  void flush() {
    if (!fixup_pending) return;
    grid_fixup_kernel<<<std::max(1u, std::min(1024u, (nb + 255) / 256)), 256, 0, stream>>>(spill, spill_n, nb,
                                                                                          cells[cur], counts);
    ++launches;
    fixup_pending = false;
  }

  void scan(StepRec* zero) {
    grid_scan_local<<<ng, 1024, 0, stream>>>(counts, nb, local, group, pw, plocal);
    grid_scan_top<<<1, 1024, 0, stream>>>(group, ng, pw, pgroup, zero);
  }

  void compact() {
    if (bitmode && !cells_valid) {  // the row straight from the planes (cells[cur] is stale)
      const uint32_t wpb = gridbits::words_per_block(wpt);
      gridbits::grid_bits_rowcount_kernel<<<nb, 256, 0, stream>>>(planes[pcur], carry[pcur], nwords, nbb, wpb,
                                                                  counts);
      scan(nullptr);
      gridbits::grid_bits_row_kernel<<<nb, 256, 0, stream>>>(planes[pcur], carry[pcur], nwords, nbb, wpb, local,
                                                             group, xs, vs);
      CKG(cudaGetLastError());
      launches += 4;
      return;
    }
    flush();
    grid_count_kernel<<<nb, kGridTPB, 0, stream>>>(cells[cur], L, counts);
    counts_valid = true;
    scan(nullptr);
    grid_compact_kernel<<<nb, kGridTPB, 0, stream>>>(cells[cur], L, local, group, xs, vs);
    CKG(cudaGetLastError());
    launches += 4;
  }

  // Folds the current row (positions, then velocities) into the device
  // digest: no transfer of the state.
  void hash_step() {
    if (!dctl) {
      CKG(cudaMalloc(&dctl, sizeof(Ctl)));
      CKG(cudaMemset(dctl, 0, sizeof(Ctl)));
      rowargs.x[0] = rowargs.x[1] = xs;
      rowargs.v[0] = rowargs.v[1] = vs;
      rowargs.n = N;
      rowargs.ctl = dctl;
    }
    compact();  // the row in rank order: xs, vs (head id 0)
    launches += digest.fold(rowargs, N, 1, stream, hash);
  }

  void pull_hash() {
    uint64_t h = 0;
    if (digest.pull(stream, &h)) hash = h;
  }

  // One step, enqueued: no host round trip (records drained in batches).
  void step() {
    if (bitmode) return step_bits();
    if (steps_done - drained >= kRecCap / 2) drain();
    const uint32_t E = mulmod(seeded(params.seed), powmod(kA, draw_exponent(steps_done, N, 0)));
    const GridArgs g{L, N, vmax, deceleration_threshold(params.p), E, 2 * powmod(kA, kGridTPB), pw, steps_done};
    if (!counts_valid) {  // after construction / set_state; later steps count as they move
      flush();
      grid_count_kernel<<<nb, kGridTPB, 0, stream>>>(cells[cur], L, counts);
      ++launches;
    }
    flush();  // the previous move's spilled cars
    scan(rec + (steps_done % kRecCap));
    if (vmax < 128)
      grid_move3_kernel<true><<<nb, kGridTPB, 0, stream>>>(cells[cur], cells[cur ^ 1], plocal, pgroup, g, rec,
                                                           counts_next, spill, spill_n);
    else
      grid_move3_kernel<false><<<nb, kGridTPB, 0, stream>>>(cells[cur], cells[cur ^ 1], plocal, pgroup, g, rec,
                                                            counts_next, spill, spill_n);
    CKG(cudaGetLastError());
    launches += 3;
    std::swap(counts, counts_next);
    counts_valid = true;
    fixup_pending = true;
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
  CKG(cudaMalloc(&d.plocal, size_t(d.nb) * 4));
  CKG(cudaMalloc(&d.pgroup, size_t(d.ng) * 4));
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
  {
    const char* force = std::getenv("NASCH_B200_GRID_BYTES");  // 1: the byte-per-cell kernels whatever vmax and L
    d.bitmode = d.vmax <= 7 && d.L % 32 == 0 && !(force && force[0] == '1');
  }
  if (d.bitmode) {
    d.nwords = d.L / 32;
    // enough blocks for a few waves of the 148 SMs before more words per thread
    d.wpt = d.nwords >= 4u * 256 * 148 * 4 ? 4 : d.nwords >= 2u * 256 * 148 * 2 ? 2 : 1;
    if (const char* w = std::getenv("NASCH_B200_GRID_WPT")) {  // 1, 2 or 4: geometry experiments and tests
      const int v = std::atoi(w);
      if (v == 1 || v == 2 || v == 4) d.wpt = v;
    }
    const uint32_t wpb = gridbits::words_per_block(d.wpt);
    d.nbb = (d.nwords + wpb - 1) / wpb;
    for (int b = 0; b < 2; ++b) {
      CKG(cudaMalloc(&d.planes[b], size_t(d.nwords) * sizeof(uint4)));
      CKG(cudaMalloc(&d.carry[b], size_t(d.nbb) * sizeof(uint4)));
    }
    CKG(cudaMalloc(&d.bcounts, size_t(d.nbb) * 4));
    CKG(cudaMalloc(&d.prank, size_t(d.nbb) * 4));
  }
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
  cudaFree(plocal);
  cudaFree(pgroup);
  cudaFree(xs);
  cudaFree(vs);
  cudaFree(rec);
  cudaFree(pw);
  cudaFree(dctl);
  for (int b = 0; b < 2; ++b) {
    cudaFree(planes[b]);
    cudaFree(carry[b]);
  }
  cudaFree(bcounts);
  cudaFree(prank);
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
  d.fixup_pending = false;  // the loaded state replaces the array
  d.planes_valid = false;
  d.cells_valid = true;
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
