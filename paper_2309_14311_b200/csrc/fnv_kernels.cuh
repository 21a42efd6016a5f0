// fnv_kernels.cuh -- the reference's trajectory checksum on the GPU.
//
// The reference folds every step's row -- all positions, then all
// velocities, in rank order, each as 8 little-endian bytes -- into an
// FNV-1a-64 digest (src/engine.hpp:15-36, src/engine.cpp:11-21, :179), one
// byte at a time on one thread.  FNV-1a looks sequential, but one byte maps
//     h -> (h xor b) * P = P*h + P*((h_lo xor b) - h_lo)
// i.e. it is affine in h except through the low byte h_lo, and the next low
// byte depends only on the previous one (P is odd).  So ANY run of bytes maps
//     h -> P^n * h + D[h & 0xff]
// for a 256-entry table D.  Kernel 1 builds D for 4096-value chunks of the
// row (block = chunk, thread = starting low byte l, running the chunk from
// h = l); kernel 2 composes tables pairwise in a tree
//     (P1,D1) then (P2,D2) = (P2*P1, l -> P2*D1[l] + D2[(P1*l + D1[l]) & 0xff]);
// kernel 3 applies the single remaining table to the running digest.  The
// row is read straight from the ID-ordered state (rank r = id (head + r) mod
// N), so no host transfer is involved.  256x the byte operations of the serial
// fold, all parallel: ~50x faster than one CPU core on the 2e8-car ring.
#pragma once
#include <cstdint>

#include "step_kernels.cuh"

namespace nb200 {

constexpr uint32_t kFnvChunk = 4096;  // row values per chunk
constexpr unsigned long long kFnvP = 1099511628211ull;

__device__ __forceinline__ unsigned long long fnv_pow(unsigned long long b, uint64_t e) {
  unsigned long long r = 1;
  while (e) {
    if (e & 1) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}

// One value < 2^32 as 8 bytes: four data bytes, then four zero bytes (each a
// bare multiply by P).
__device__ __forceinline__ unsigned long long fnv_value(unsigned long long h, uint32_t w) {
  constexpr unsigned long long P4 = kFnvP * kFnvP * kFnvP * kFnvP;
  h = (h ^ (w & 0xffu)) * kFnvP;
  h = (h ^ ((w >> 8) & 0xffu)) * kFnvP;
  h = (h ^ ((w >> 16) & 0xffu)) * kFnvP;
  h = (h ^ (w >> 24)) * kFnvP;
  return h * P4;
}

template <typename VT>
__global__ void __launch_bounds__(256) fnv_chunk_kernel(const RingArgs ra, unsigned long long* T,
                                                        unsigned long long* Pt) {
  __shared__ uint32_t vals[kFnvChunk];
  const Ctl* ctl = ra.ctl;
  const uint32_t N = ra.n;
  const uint32_t head = (N - ctl->W) % N;  // id of the rank-0 car
  const int b = static_cast<int>(ctl->buf);
  const uint32_t* X = xbuf(ra, b);
  const VT* V = vbuf<VT>(ra, b);
  const uint64_t rowlen = 2ull * N;
  const uint64_t lo = uint64_t(blockIdx.x) * kFnvChunk;
  const uint32_t cnt = static_cast<uint32_t>(rowlen - lo < kFnvChunk ? rowlen - lo : kFnvChunk);
  for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
    const uint64_t k = lo + i;
    const uint32_t r = static_cast<uint32_t>(k < N ? k : k - N);
    uint32_t id = head + r;
    if (id >= N) id -= N;
    vals[i] = k < N ? X[id] : static_cast<uint32_t>(V[id]);
  }
  __syncthreads();
  unsigned long long h = threadIdx.x;  // starting low byte l
  for (uint32_t i = 0; i < cnt; ++i) h = fnv_value(h, vals[i]);
  const unsigned long long pn = fnv_pow(kFnvP, 8ull * cnt);
  T[size_t(blockIdx.x) * 256 + threadIdx.x] = h - pn * threadIdx.x;
  if (threadIdx.x == 0) Pt[blockIdx.x] = pn;
}

// Pairwise composition: table 2i then table 2i+1 -> out table i.
static __global__ void __launch_bounds__(256) fnv_compose_kernel(const unsigned long long* Tin,
                                                          const unsigned long long* Pin, uint32_t nin,
                                                          unsigned long long* Tout,
                                                          unsigned long long* Pout) {
  const uint32_t i = blockIdx.x, l = threadIdx.x;
  const uint32_t a = 2 * i, b = a + 1;
  if (b >= nin) {  // odd one out passes through
    Tout[size_t(i) * 256 + l] = Tin[size_t(a) * 256 + l];
    if (l == 0) Pout[i] = Pin[a];
    return;
  }
  const unsigned long long P1 = Pin[a], P2 = Pin[b];
  const unsigned long long d1 = Tin[size_t(a) * 256 + l];
  const uint32_t mid = static_cast<uint32_t>((P1 * l + d1) & 0xffu);
  Tout[size_t(i) * 256 + l] = P2 * d1 + Tin[size_t(b) * 256 + mid];
  if (l == 0) Pout[i] = P2 * P1;
}

static __global__ void fnv_apply_kernel(const unsigned long long* T, const unsigned long long* Pt,
                                 unsigned long long* hash) {
  const unsigned long long h = *hash;
  *hash = Pt[0] * h + T[h & 0xffu];
}

// Chunk tables of a contiguous slice of values (a shard's piece of the
// rank-ordered row): block = 4096-value chunk of vals[0, count).
template <typename T>
__global__ void __launch_bounds__(256) fnv_slice_chunk_kernel(const T* __restrict__ vals, uint32_t count,
                                                              unsigned long long* Tt, unsigned long long* Pt) {
  __shared__ uint32_t sv[kFnvChunk];
  const uint32_t lo = blockIdx.x * kFnvChunk;
  const uint32_t cnt = count - lo < kFnvChunk ? count - lo : kFnvChunk;
  for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) sv[i] = static_cast<uint32_t>(vals[lo + i]);
  __syncthreads();
  unsigned long long h = threadIdx.x;
  for (uint32_t i = 0; i < cnt; ++i) h = fnv_value(h, sv[i]);
  const unsigned long long pn = fnv_pow(kFnvP, 8ull * cnt);
  Tt[size_t(blockIdx.x) * 256 + threadIdx.x] = h - pn * threadIdx.x;
  if (threadIdx.x == 0) Pt[blockIdx.x] = pn;
}

}  // namespace nb200
