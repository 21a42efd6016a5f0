// grid_bits.cuh -- the cell-array engine (src/model.cpp:99-129) in bit planes,
// for vmax <= 7 and L a multiple of 32: 32 cells per uint4 {occupied, v bit 0,
// v bit 1, v bit 2}, half a byte per cell instead of one, and the whole rule
// but the draws evaluated for 32 cells at once with bitwise operations
// ("multi-spin coding"):
//   gap >= d        F_d = ~(occ >> 1) & ... & ~(occ >> d) (funnel shifts across
//                   the next word: the lookahead is at most vmax cells)
//   min(v+1, vmax, gap) >= d     T_{d-1} & F_d, T_d = cars with v >= d
//                   (thermometer form from the three binary planes)
//   random slowdown v' >= d      vc_{d+1} | (vc_d & ~dec)
//   move            cars with v' = d exactly shifted up d cells; the bits that
//                   leave the word go to the next word (register, shuffle,
//                   shared memory, or the block's carry word in HBM, which the
//                   next block ORs into its first word when it loads it next
//                   step -- no fixup pass)
// Only the draws are per car: rank order is ascending bit order, so a thread
// walks the set bits of its words with Q <- Q a (one mulmod_x2 per car) from
// Q = E a^(rank of its first car), the rank from the block scan of popcounts.
// The velocity sum is the sum of the thermometer popcounts, the wrap count the
// popcount of the last word's overflow.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "minstd.hpp"
#include "step_kernels.cuh"

namespace nb200 {
namespace gridbits {

constexpr int kTPB = 256;
// 32-cell words per thread (WPT): 4 on large rings (the per-thread fixed work
// -- scan, draw base, seams -- amortised over more cells; measured 46 -> 41 us
// per step at L = 1e8 against 2), 2 and 1 on smaller ones for enough blocks.
__host__ __device__ constexpr uint32_t words_per_block(int wpt) { return static_cast<uint32_t>(kTPB * wpt); }

struct BitArgs {
  uint32_t nwords;     // L / 32
  uint32_t tp;         // deceleration threshold
  uint32_t E;          // s0 a^(t N + 1)
  uint32_t a2;         // 2 a
  uint32_t one, two;   // 1 and 2 as launch parameters: keep the compare IMADs (FMA pipe; the kernel is ALU-pipe bound)
  uint32_t p2[8];      // 2^d, likewise
  uint32_t apw[8];     // a^k
  uint32_t ainv[8];    // a^-k
  const uint32_t* pw;  // [3][4096]: a^j, a^(4096 j), a^(4096^2 j)
  unsigned long long t;
};

// Cars with velocity >= D from the binary planes (D = 0: every car).
template <int D>
__device__ __forceinline__ uint32_t thermo(uint32_t o, uint32_t p0, uint32_t p1, uint32_t p2) {
  if constexpr (D == 0) return o;
  if constexpr (D == 1) return p0 | p1 | p2;
  if constexpr (D == 2) return p1 | p2;
  if constexpr (D == 3) return p2 | (p1 & p0);
  if constexpr (D == 4) return p2;
  if constexpr (D == 5) return p2 & (p0 | p1);
  if constexpr (D == 6) return p2 & p1;
  return p2 & p1 & p0;
}

// One word: the new velocities' thermometer masks vp[1..VMAX] from the word,
// the next word's occupancy and the deceleration mask.
template <int VMAX>
__device__ __forceinline__ void word_rule(uint32_t o, uint32_t p0, uint32_t p1, uint32_t p2, uint32_t nx,
                                          uint32_t (&vc)[VMAX + 2]) {
  uint32_t F = 0xffffffffu;
  vc[0] = o;
  vc[VMAX + 1] = 0;
#pragma unroll
  for (int d = 1; d <= VMAX; ++d) {
    F &= ~__funnelshift_r(o, nx, d);  // cell i + d empty, for every i at once
    uint32_t T;
    switch (d - 1) {
      case 0: T = thermo<0>(o, p0, p1, p2); break;
      case 1: T = thermo<1>(o, p0, p1, p2); break;
      case 2: T = thermo<2>(o, p0, p1, p2); break;
      case 3: T = thermo<3>(o, p0, p1, p2); break;
      case 4: T = thermo<4>(o, p0, p1, p2); break;
      case 5: T = thermo<5>(o, p0, p1, p2); break;
      default: T = thermo<6>(o, p0, p1, p2); break;
    }
    vc[d] = T & F;  // min(v + 1, vmax, gap) >= d
  }
}

// a^r from the three power tables pw = [a^j, a^(4096 j), a^(4096^2 j)], j < 4096.
__device__ __forceinline__ uint32_t apow3(const uint32_t* pw, uint32_t r) {
  return mulmod(mulmod(__ldg(pw + (r & 4095u)), __ldg(pw + 4096 + ((r >> 12) & 4095u))),
                __ldg(pw + 8192 + (r >> 24)));
}

// The exclusive scan of the blocks' car counts by ONE block of kTPB threads:
// prank[b] = a^(rank of block b's first car), a block's cars being those in
// its words plus the ones the previous block carried over its end.  Runs
// after a pack only (the moves keep prank current themselves, below).
// Thread t scans a contiguous range of blocks.
__device__ __forceinline__ void scan_blocks(const uint32_t* counts, const uint4* carry, uint32_t nbb,
                                            const uint32_t* __restrict__ pw, uint32_t* prank, uint32_t* s_scan) {
  constexpr int B = 16;  // entries in flight per thread: the loads of a batch are independent
  const uint32_t per = (nbb + kTPB - 1) / kTPB;
  const uint32_t i0 = min(threadIdx.x * per, nbb), i1 = min(i0 + per, nbb);
  uint32_t sum = 0;
  for (uint32_t base = i0; base < i1; base += B) {
    uint32_t c[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const uint32_t i = base + j;
      c[j] = i < i1 ? __ldcg(counts + i) + __popc(__ldcg(&carry[(i ? i : nbb) - 1].x)) : 0u;
    }
#pragma unroll
    for (int j = 0; j < B; ++j) sum += c[j];
  }
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t incl = sum;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, incl, s);
    if (lane >= static_cast<uint32_t>(s)) incl += n;
  }
  if (lane == 31) s_scan[warp] = incl;
  __syncthreads();
  uint32_t r = incl - sum;
  for (uint32_t w = 0; w < warp; ++w) r += s_scan[w];
  for (uint32_t base = i0; base < i1; base += B) {
    uint32_t c[B], rr[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const uint32_t i = base + j;
      c[j] = i < i1 ? __ldcg(counts + i) + __popc(__ldcg(&carry[(i ? i : nbb) - 1].x)) : 0u;
    }
#pragma unroll
    for (int j = 0; j < B; ++j) {
      rr[j] = r;
      r += c[j];
    }
#pragma unroll
    for (int j = 0; j < B; ++j)
      if (base + j < i1) prank[base + j] = apow3(pw, rr[j]);
  }
}

__global__ void __launch_bounds__(kTPB) grid_bits_scan_kernel(const uint32_t* counts, const uint4* carry,
                                                              uint32_t nbb, const uint32_t* pw, uint32_t* prank,
                                                              StepRec* zero) {
  __shared__ uint32_t s_scan[kTPB / 32];
  scan_blocks(counts, carry, nbb, pw, prank, s_scan);
  if (threadIdx.x == 0) {
    zero->sumv = 0;
    zero->c = 0;
  }
}

// The move of one step over the bit planes.  Block b owns words
// [b kWordsPerBlock, ...), thread t the kWPT consecutive words from
// (b kTPB + t) kWPT.  PARTIAL: the ring's last block when it is not whole
// (dead words read as empty, the last live word anywhere in the block).
template <int VMAX, int kWPT, bool PARTIAL>
__device__ __forceinline__ void bitmove_block(const uint4* __restrict__ in, uint4* __restrict__ out,
                                              const uint4* __restrict__ carry_in, uint4* __restrict__ carry_out,
                                              uint32_t* prank, const BitArgs& g, StepRec* rec, uint32_t* s_cnt,
                                              uint32_t* s_first, uint32_t* s_hi) {
  constexpr int NW = kTPB / 32;
  constexpr uint32_t kWordsPerBlock = words_per_block(kWPT);
  const uint32_t b = blockIdx.x, nbb = gridDim.x;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t w0 = (b * kTPB + threadIdx.x) * kWPT;
  const uint32_t lastw = PARTIAL ? g.nwords - 1u : (b + 1) * kWordsPerBlock - 1u;  // the block's last live word
  const bool has_last = PARTIAL ? (w0 <= lastw && lastw < w0 + kWPT) : threadIdx.x == kTPB - 1;
  // every global load first
  uint32_t o[kWPT], p0[kWPT], p1[kWPT], p2[kWPT];
#pragma unroll
  for (int k = 0; k < kWPT; ++k) {
    uint4 u = make_uint4(0, 0, 0, 0);
    if (!PARTIAL || w0 + k <= lastw) u = __ldg(in + w0 + k);
    o[k] = u.x; p0[k] = u.y; p1[k] = u.z; p2[k] = u.w;
  }
  uint32_t nxt_global = 0;
  if (has_last) {  // the first word after the block (cyclic), with the cars carried into it last step
    const uint32_t wn = b + 1 == nbb ? 0u : (b + 1) * kWordsPerBlock;
    nxt_global = __ldg(in + wn).x | __ldg(carry_in + b).x;
  }
  const uint4 cprev = __ldg(carry_in + (b + nbb - 1) % nbb);  // the cars the previous block carried over its end
  const uint32_t wrapped = __popc(__ldg(carry_in + nbb - 1).x);
  if (threadIdx.x == 0) {
    o[0] |= cprev.x; p0[0] |= cprev.y; p1[0] |= cprev.z; p2[0] |= cprev.w;
  }
  // a^(rank of the block's first car): last step's, times a^wrapped a^-carried
  const uint32_t pr = mulmod_d(mulmod_d(__ldcg(prank + b), g.apw[wrapped]), g.ainv[__popc(cprev.x)]);
  // ranks: block scan of the popcounts
  uint32_t cnt = 0;
#pragma unroll
  for (int k = 0; k < kWPT; ++k) cnt += __popc(o[k]);
  uint32_t incl = cnt;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, incl, s);
    if (lane >= static_cast<uint32_t>(s)) incl += n;
  }
  if (lane == 31) s_cnt[warp] = incl;
  if (lane == 0) s_first[warp] = o[0];
  __syncthreads();
  const uint32_t cw = lane < static_cast<uint32_t>(NW) ? s_cnt[lane] : 0u;
  const uint32_t wbase = __reduce_add_sync(0xffffffffu, lane < warp ? cw : 0u);
  const uint32_t j0 = wbase + incl - cnt;  // block-local rank of this thread's first car
  uint32_t nxt_thread = __shfl_down_sync(0xffffffffu, o[0], 1);
  if (lane == 31) nxt_thread = warp + 1 < static_cast<uint32_t>(NW) ? s_first[warp + 1] : nxt_global;
  const uint32_t Eb = mulmod_d(g.E, pr);  // E a^(rank of the block's first car)
  uint32_t Q = mulmod_d(mulmod_d(Eb, __ldg(g.pw + (j0 & 4095u))), __ldg(g.pw + 4096 + (j0 >> 12)));

  uint32_t no[kWPT], n0[kWPT], n1[kWPT], n2[kWPT];  // the next array's words
  uint32_t ho = 0, h0 = 0, h1 = 0, h2 = 0;          // bits leaving the previous word
  uint32_t co = 0, c0 = 0, c1 = 0, c2 = 0;          // ... leaving the block's last word
  uint32_t sumv = 0;
  const uint32_t ntp = 0u - g.tp;
#pragma unroll
  for (int k = 0; k < kWPT; ++k) {
    uint32_t nx = k + 1 < kWPT ? o[k + 1 < kWPT ? k + 1 : k] : nxt_thread;
    if (PARTIAL && w0 + k == lastw) nx = nxt_global;
    uint32_t vc[VMAX + 2];
    word_rule<VMAX>(o[k], p0[k], p1[k], p2[k], nx, vc);
    // The draws, one per car in ascending cell order (model.cpp:51: always
    // consumed).  s < tp as bit 31 of s - tp (both below 2^31), moved to bit 0
    // by a multiply-high and selected by a multiply-add: three FMA-pipe
    // instructions (1 and 2 are launch parameters so that they stay IMADs)
    // instead of ISETP + SEL + LOP3 on the ALU pipe, which bounds the kernel.
    uint32_t dec = 0;
    for (uint32_t m = o[k]; m;) {
      const uint32_t s = Q;
      Q = mulmod_x2(g.a2, Q);
      uint32_t lt;
      asm("{ .reg .u32 t; mad.lo.u32 t, %1, %2, %3; mul.hi.u32 %0, t, %4; }"
          : "=r"(lt) : "r"(s), "r"(g.one), "r"(ntp), "r"(g.two));
      const uint32_t bit = m & (0u - m);
      dec += lt * bit;
      m ^= bit;
    }
    uint32_t lo_o, lo_0 = 0, lo_1 = 0, lo_2 = 0, hi_o = 0, hi_0 = 0, hi_1 = 0, hi_2 = 0;
    uint32_t vnext = 0;  // v' >= d + 1
    uint32_t stay = 0;
#pragma unroll
    for (int d = VMAX; d >= 1; --d) {
      const uint32_t vp = vc[d + 1] | (vc[d] & ~dec);  // v' >= d
      sumv += __popc(vp);
      const uint32_t X = vp & ~vnext;  // v' == d
      vnext = vp;
      // X >> (32 - d) as the high word of X 2^d (2^d a launch parameter: an
      // IMAD.HI on the FMA pipe, not a shift on the ALU pipe)
      const uint32_t l = X << d, h = __umulhi(X, g.p2[d]);
      stay |= l;
      hi_o |= h;
      if (d & 1) { lo_0 |= l; hi_0 |= h; }
      if (d & 2) { lo_1 |= l; hi_1 |= h; }
      if (d & 4) { lo_2 |= l; hi_2 |= h; }
    }
    lo_o = stay | (o[k] & ~vnext);  // v' == 0 stays
    no[k] = lo_o | ho; n0[k] = lo_0 | h0; n1[k] = lo_1 | h1; n2[k] = lo_2 | h2;
    ho = hi_o; h0 = hi_0; h1 = hi_1; h2 = hi_2;
    if (PARTIAL && w0 + k == lastw) { co = hi_o; c0 = hi_0; c1 = hi_1; c2 = hi_2; }
  }
  if (!PARTIAL) { co = ho; c0 = h0; c1 = h1; c2 = h2; }  // read by the has_last thread only
  // the last word's overflow to the next thread's first word (<= 7 bits a plane)
  const uint32_t pk = ho | (h0 << 7) | (h1 << 14) | (h2 << 21);
  uint32_t pin = __shfl_up_sync(0xffffffffu, pk, 1);
  if (lane == 31) s_hi[warp] = pk;
  __syncthreads();
  if (lane == 0) pin = warp ? s_hi[warp - 1] : 0u;
  no[0] |= pin & 0x7fu; n0[0] |= (pin >> 7) & 0x7fu; n1[0] |= (pin >> 14) & 0x7fu; n2[0] |= (pin >> 21) & 0x7fu;
#pragma unroll
  for (int k = 0; k < kWPT; ++k)
    if (!PARTIAL || w0 + k <= lastw) out[w0 + k] = make_uint4(no[k], n0[k], n1[k], n2[k]);
  sumv = __reduce_add_sync(0xffffffffu, sumv);
  if (lane == 0 && sumv) atomicAdd(&rec[g.t % kRecCap].sumv, static_cast<unsigned long long>(sumv));
  if (has_last) {
    carry_out[b] = make_uint4(co, c0, c1, c2);
    if (b + 1 == nbb && co) atomicAdd(&rec[g.t % kRecCap].c, static_cast<unsigned int>(__popc(co)));
  }
  if (threadIdx.x == 0) {
    prank[b] = pr;
    if (b == 0) {  // the next step's record
      StepRec* nr = rec + ((g.t + 1) % kRecCap);
      nr->sumv = 0;
      nr->c = 0;
    }
  }
}

// One step is ONE launch.  No scan between steps: cars never overtake, so the
// rank of a block's first car changes from one step to the next by the cars
// that wrapped past the ring's end (they take the lowest ranks) minus the
// cars the previous block carried over this block's start (they precede the
// block's own cars) -- both are popcounts of last step's carry words, which
// the block reads anyway.  Each block keeps a^(its rank) in prank[b] and
// advances it by a^wrapped a^-carried.
template <int VMAX, int WPT>
__global__ void __launch_bounds__(kTPB, WPT == 4 ? 5 : 1) grid_bitmove_kernel(const uint4* __restrict__ in, uint4* __restrict__ out,
                                                            const uint4* __restrict__ carry_in,
                                                            uint4* __restrict__ carry_out, uint32_t* prank,
                                                            BitArgs g, StepRec* rec) {
  constexpr int NW = kTPB / 32;
  __shared__ uint32_t s_cnt[NW], s_first[NW + 1], s_hi[NW];
  if ((blockIdx.x + 1) * words_per_block(WPT) <= g.nwords)
    bitmove_block<VMAX, WPT, false>(in, out, carry_in, carry_out, prank, g, rec, s_cnt, s_first, s_hi);
  else
    bitmove_block<VMAX, WPT, true>(in, out, carry_in, carry_out, prank, g, rec, s_cnt, s_first, s_hi);
}

// cells (one byte per cell, 0xff = empty) -> planes; one thread per word.
__global__ void grid_pack_kernel(const uint8_t* __restrict__ cells, uint32_t nwords, uint4* __restrict__ planes) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nwords) return;
  const uint4* src = reinterpret_cast<const uint4*>(cells) + 2 * size_t(i);
  const uint4 a = src[0], c = src[1];
  const uint32_t ws[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
  uint32_t o = 0, q0 = 0, q1 = 0, q2 = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint32_t w = ws[q];
    o |= (((__vcmpne4(w, 0xffffffffu) & 0x01010101u) * 0x01020408u) >> 24) << (4 * q);
    q0 |= (((w & 0x01010101u) * 0x01020408u) >> 24) << (4 * q);
    q1 |= ((((w >> 1) & 0x01010101u) * 0x01020408u) >> 24) << (4 * q);
    q2 |= ((((w >> 2) & 0x01010101u) * 0x01020408u) >> 24) << (4 * q);
  }
  planes[i] = make_uint4(o, q0 & o, q1 & o, q2 & o);
}

// The readers' rank-ordered row (state, frames, checksum) straight from the
// planes, in 256-word (8192-cell) blocks like the byte form's compaction:
// a word's cars are its own plus, for the first word of a move block, the
// cars the previous move block carried over its end (still in `carry`).
__device__ __forceinline__ uint4 word_with_carry(const uint4* __restrict__ planes, const uint4* __restrict__ carry,
                                                 uint32_t w, uint32_t nbb, uint32_t wpb) {
  uint4 u = planes[w];
  if (w % wpb == 0) {
    const uint4 c = carry[(w / wpb + nbb - 1) % nbb];
    u.x |= c.x; u.y |= c.y; u.z |= c.z; u.w |= c.w;
  }
  return u;
}

__global__ void __launch_bounds__(256) grid_bits_rowcount_kernel(const uint4* __restrict__ planes,
                                                                 const uint4* __restrict__ carry, uint32_t nwords,
                                                                 uint32_t nbb, uint32_t wpb, uint32_t* counts) {
  __shared__ uint32_t s[8];
  const uint32_t w = blockIdx.x * 256u + threadIdx.x;
  uint32_t c = w < nwords ? __popc(word_with_carry(planes, carry, w, nbb, wpb).x) : 0u;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x / 32] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int k = 0; k < 8; ++k) t += s[k];
    counts[blockIdx.x] = t;
  }
}

// local/group: the two-level exclusive scan of the row counts (grid.cu).
__global__ void __launch_bounds__(256) grid_bits_row_kernel(const uint4* __restrict__ planes,
                                                            const uint4* __restrict__ carry, uint32_t nwords,
                                                            uint32_t nbb, uint32_t wpb,
                                                            const uint32_t* __restrict__ local,
                                                            const uint32_t* __restrict__ group, uint32_t* xs,
                                                            uint8_t* vs) {
  __shared__ uint32_t s_w[8];
  const uint32_t w = blockIdx.x * 256u + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint4 u = make_uint4(0, 0, 0, 0);
  if (w < nwords) u = word_with_carry(planes, carry, w, nbb, wpb);
  const uint32_t cnt = __popc(u.x);
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += n;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  uint32_t r = local[blockIdx.x] + group[blockIdx.x >> 10] + incl - cnt;
  for (uint32_t k = 0; k < warp; ++k) r += s_w[k];
  for (uint32_t m = u.x; m; m &= m - 1u) {
    const uint32_t pos = __ffs(m) - 1u;
    xs[r] = w * 32u + pos;
    vs[r] = static_cast<uint8_t>(((u.y >> pos) & 1u) | (((u.z >> pos) & 1u) << 1) | (((u.w >> pos) & 1u) << 2));
    ++r;
  }
}

// Cars per block of kTPB wpt words.
__global__ void __launch_bounds__(kTPB) grid_bitcount_kernel(const uint4* __restrict__ planes, uint32_t nwords,
                                                             uint32_t wpt, uint32_t* counts) {
  __shared__ uint32_t s[kTPB / 32];
  uint32_t c = 0;
  for (uint32_t k = 0; k < wpt; ++k) {
    const uint32_t w = (blockIdx.x * kTPB + threadIdx.x) * wpt + k;
    if (w < nwords) c += __popc(planes[w].x);
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x / 32] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kTPB / 32; ++w) t += s[w];
    counts[blockIdx.x] = t;
  }
}

}  // namespace gridbits
}  // namespace nb200
