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


// ---- low-byte decomposition of the row digest (GpuRing) -------------------
//
// The 256-start tables above do the 64-bit FNV work 256 times over.  But the
// only thing a chunk's result needs from the incoming state is its low byte,
// and the low byte evolves on its own: l -> ((l ^ b) * P) mod 256, with
// P mod 256 = 0xb3.  So a step's digest is computed in three passes:
//   A  (fnv_map8_kernel)   per 2048-value chunk, the 8-bit map l_in -> l_out
//                          of its low byte, for all 256 starts at once: two
//                          starts per 32-bit register (16-bit lanes, masked
//                          to 8 bits before each multiply: LOP3 + IMAD per
//                          byte for two starts), and only 128 starts tracked
//                          since the map commutes with flipping bit 7
//                          (F(l ^ 0x80) = F(l) ^ 0x80: both ops carry bit 7
//                          straight through);
//   B  (fnv_group8_kernel, fnv_walk8_kernel)  the maps composed 256 at a time
//                          up a tree, then walked down from the digest's
//                          known low byte: every chunk's incoming low byte;
//   C  (fnv_affine_kernel) each chunk once, in exact 64-bit arithmetic, from
//                          that low byte: h -> P^(8n) h + d_c; the chunks'
//                          affine maps reduced in a tree (fnv_affine_reduce)
//                          and applied to the running digest.
// Pass A does 1/2 of the byte work of the old tables in 8-bit lanes instead
// of 64-bit products; pass C does the 64-bit work once.
constexpr uint32_t kFnvRowChunk = 2048;  // row values per chunk
constexpr uint32_t kFnvP8 = 0xb3u;       // P mod 256
constexpr uint32_t kFnvP8_5 = (kFnvP8 * kFnvP8 * kFnvP8 * kFnvP8 * kFnvP8) & 0xffu;  // a value's last byte + 4 zero bytes
constexpr uint32_t kFnvP8_8 = (kFnvP8_5 * kFnvP8 * kFnvP8 * kFnvP8) & 0xffu;       // a < 256 value: 1 byte + 7 zero bytes
constexpr int kMap8Warps = 8;
constexpr uint32_t kFnvSubs = 4;                          // pass C threads per chunk
constexpr uint32_t kFnvSubLen = kFnvRowChunk / kFnvSubs;  // 512 values each

// Row value k of the current step (k < N: position of rank k, else the
// velocity of rank k - N; rank r is id (head + r) mod N).
template <typename VT>
__device__ __forceinline__ uint32_t fnv_row_value(const uint32_t* X, const VT* V, uint32_t N, uint32_t head,
                                                  uint64_t k) {
  const bool pos = k < N;
  const uint32_t r = static_cast<uint32_t>(pos ? k : k - N);
  uint32_t id = head + r;
  if (id >= N) id -= N;
  return pos ? __ldg(X + id) : static_cast<uint32_t>(__ldg(V + id));
}

// Pass A: one warp per chunk.  Lane t tracks starts t, t+32 (one register)
// and t+64, t+96 (another).  Out: F[c][l], 256 bytes per chunk.
template <typename VT>
__global__ void __launch_bounds__(32 * kMap8Warps) fnv_map8_kernel(const RingArgs ra, uint8_t* F, uint8_t* Fsub,
                                                                   uint32_t nchunks) {
  __shared__ uint4 s_bb[kMap8Warps][32];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t c = blockIdx.x * kMap8Warps + warp;
  if (c >= nchunks) return;
  const Ctl* ctl = ra.ctl;
  const uint32_t N = ra.n;
  const uint32_t head = (N - ctl->W) % N;
  const int b = static_cast<int>(ctl->buf);
  const uint32_t* X = xbuf(ra, b);
  const VT* V = vbuf<VT>(ra, b);
  const uint64_t rowlen = 2ull * N;
  const uint64_t k0 = uint64_t(c) * kFnvRowChunk;
  const uint32_t cnt = static_cast<uint32_t>(rowlen - k0 < kFnvRowChunk ? rowlen - k0 : kFnvRowChunk);
  constexpr uint32_t M = 0x00ff00ffu;
  uint32_t h0 = lane | ((lane + 32u) << 16), h1 = (lane + 64u) | ((lane + 96u) << 16);
  for (uint32_t base = 0; base < cnt; base += 32) {
    if (base + lane < cnt) {
      const uint32_t w = fnv_row_value<VT>(X, V, N, head, k0 + base + lane);
      s_bb[warp][lane] = make_uint4(__byte_perm(w, 0u, 0x4040u), __byte_perm(w, 0u, 0x4141u),
                                    __byte_perm(w, 0u, 0x4242u), __byte_perm(w, 0u, 0x4343u));
    }
    __syncwarp();
    const uint32_t n32 = cnt - base < 32u ? cnt - base : 32u;
    // positions (and any velocity >= 256): four data bytes, then four zero
    // bytes folded into the last multiply; u8 velocities: one byte + seven
    const uint64_t kb = k0 + base;
    const uint32_t npos = kb >= N ? 0u : (kb + n32 <= N ? n32 : static_cast<uint32_t>(N - kb));
    const uint32_t nfull = sizeof(VT) == 1 ? npos : n32;
    auto full = [&](uint32_t j) {
      const uint4 bb = s_bb[warp][j];
      h0 = ((h0 ^ bb.x) & M) * kFnvP8;
      h1 = ((h1 ^ bb.x) & M) * kFnvP8;
      h0 = ((h0 ^ bb.y) & M) * kFnvP8;
      h1 = ((h1 ^ bb.y) & M) * kFnvP8;
      h0 = ((h0 ^ bb.z) & M) * kFnvP8;
      h1 = ((h1 ^ bb.z) & M) * kFnvP8;
      h0 = ((h0 ^ bb.w) & M) * kFnvP8_5;
      h1 = ((h1 ^ bb.w) & M) * kFnvP8_5;
    };
    auto one = [&](uint32_t j) {
      const uint32_t bx = s_bb[warp][j].x;
      h0 = ((h0 ^ bx) & M) * kFnvP8_8;
      h1 = ((h1 ^ bx) & M) * kFnvP8_8;
    };
    if (nfull == 32) {  // the common case, unrolled
#pragma unroll
      for (uint32_t j = 0; j < 32; ++j) full(j);
    } else if (nfull == 0 && n32 == 32) {
#pragma unroll
      for (uint32_t j = 0; j < 32; ++j) one(j);
    } else {
      for (uint32_t j = 0; j < nfull; ++j) full(j);
      for (uint32_t j = nfull; j < n32; ++j) one(j);
    }
    __syncwarp();
    // the map from the chunk's start to each sub-chunk boundary (pass C
    // runs kFnvSubs threads per chunk from these)
    const uint32_t done = base + n32;
    if (done % kFnvSubLen == 0 && done < cnt) {
      uint8_t* sub = Fsub + (size_t(c) * (kFnvSubs - 1) + done / kFnvSubLen - 1) * 256;
      const uint32_t g[4] = {h0 & 0xffu, (h0 >> 16) & 0xffu, h1 & 0xffu, (h1 >> 16) & 0xffu};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        sub[lane + 32u * q] = static_cast<uint8_t>(g[q]);
        sub[(lane + 32u * q) ^ 0x80u] = static_cast<uint8_t>(g[q] ^ 0x80u);
      }
    }
  }
  uint8_t* out = F + size_t(c) * 256;
  const uint32_t f[4] = {h0 & 0xffu, (h0 >> 16) & 0xffu, h1 & 0xffu, (h1 >> 16) & 0xffu};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t s = lane + 32u * q;
    out[s] = static_cast<uint8_t>(f[q]);
    out[s ^ 0x80u] = static_cast<uint8_t>(f[q] ^ 0x80u);
  }
}

// Pass B, up: block g composes maps [256 g, 256 g + 256) of `in` (n maps)
// into out[g]: thread l follows start l through them (maps staged in
// shared memory).
static __global__ void __launch_bounds__(256) fnv_group8_kernel(const uint8_t* in, uint32_t n, uint8_t* out) {
  extern __shared__ uint8_t s_maps[];  // [256][256]
  const uint32_t g = blockIdx.x;
  const uint32_t m = n - 256u * g < 256u ? n - 256u * g : 256u;
  const uint4* src = reinterpret_cast<const uint4*>(in + size_t(g) * 256 * 256);
  uint4* dst = reinterpret_cast<uint4*>(s_maps);
  for (uint32_t i = threadIdx.x; i < m * 16u; i += 256) dst[i] = src[i];
  __syncthreads();
  uint32_t l = threadIdx.x;
  for (uint32_t i = 0; i < m; ++i) l = s_maps[i * 256u + l];
  out[size_t(g) * 256 + threadIdx.x] = static_cast<uint8_t>(l);
}

// Pass B, down: block g knows the low byte entering its group (lb_in[g], or
// the digest's low byte at the top) and walks its <= 256 maps, writing the
// low byte entering each (lb_out[256 g + i]).
static __global__ void __launch_bounds__(256) fnv_walk8_kernel(const uint8_t* maps, uint32_t n, const uint8_t* lb_in,
                                                        const unsigned long long* hash, uint8_t* lb_out) {
  extern __shared__ uint8_t s_maps[];  // [256][256]
  const uint32_t g = blockIdx.x;
  const uint32_t m = n - 256u * g < 256u ? n - 256u * g : 256u;
  const uint4* src = reinterpret_cast<const uint4*>(maps + size_t(g) * 256 * 256);
  uint4* dst = reinterpret_cast<uint4*>(s_maps);
  for (uint32_t i = threadIdx.x; i < m * 16u; i += 256) dst[i] = src[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t l = lb_in ? lb_in[g] : static_cast<uint32_t>(*hash & 0xffu);
    for (uint32_t i = 0; i < m; ++i) {
      lb_out[256u * g + i] = static_cast<uint8_t>(l);
      l = s_maps[i * 256u + l];
    }
  }
}

// Pass C: one thread per sub-chunk (kFnvSubLen values) runs the exact
// 64-bit FNV of its values from the 64-bit state lb (its true incoming low
// byte, upper bytes 0; a chunk's later sub-chunks read theirs from the
// cumulative sub-chunk maps of pass A): h_out = P^(8n) lb + d, so the
// sub-chunk maps the true state h to P^(8n) h + d.  Values staged through
// shared memory 32 per sub-chunk at a time (coalesced loads, all in flight
// before the stores; rows padded against bank conflicts).
constexpr int kAffTPB = 128;
template <typename VT>
__global__ void __launch_bounds__(kAffTPB) fnv_affine_kernel(const RingArgs ra, const uint8_t* lb, const uint8_t* Fsub,
                                                             uint32_t nsub, unsigned long long* A,
                                                             unsigned long long* D) {
  __shared__ uint32_t s_v[kAffTPB][33];
  const Ctl* ctl = ra.ctl;
  const uint32_t N = ra.n;
  const uint32_t head = (N - ctl->W) % N;
  const int b = static_cast<int>(ctl->buf);
  const uint32_t* X = xbuf(ra, b);
  const VT* V = vbuf<VT>(ra, b);
  const uint64_t rowlen = 2ull * N;
  const uint32_t s0 = blockIdx.x * kAffTPB;
  const uint32_t s = s0 + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  constexpr unsigned long long P4 = kFnvP * kFnvP * kFnvP * kFnvP;
  unsigned long long h = 0;
  uint32_t cnt = 0;
  if (s < nsub) {
    const uint32_t c = s / kFnvSubs, q = s % kFnvSubs;
    const uint32_t l = lb[c];
    h = q == 0 ? l : Fsub[(size_t(c) * (kFnvSubs - 1) + q - 1) * 256 + l];
    const uint64_t k0 = uint64_t(s) * kFnvSubLen;
    cnt = static_cast<uint32_t>(rowlen - k0 < kFnvSubLen ? rowlen - k0 : kFnvSubLen);
  }
  const unsigned long long h_in = h;
  for (uint32_t t = 0; t < kFnvSubLen; t += 32) {
    constexpr int kRows = kAffTPB / (kAffTPB / 32);
    uint32_t vals[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const uint32_t sr = s0 + warp + r * (kAffTPB / 32);
      const uint64_t k = uint64_t(sr) * kFnvSubLen + t + lane;
      vals[r] = (sr < nsub && k < rowlen) ? fnv_row_value<VT>(X, V, N, head, k) : 0u;
    }
#pragma unroll
    for (int r = 0; r < kRows; ++r) s_v[warp + r * (kAffTPB / 32)][lane] = vals[r];
    __syncthreads();
    const uint32_t m = cnt > t ? (cnt - t < 32u ? cnt - t : 32u) : 0u;
    for (uint32_t i = 0; i < m; ++i) {
      const uint32_t w = s_v[threadIdx.x][i];
      if (w < 256u) {  // velocities (and tiny positions): one data byte
        h = (h ^ w) * kFnvP;
        h *= P4 * kFnvP * kFnvP * kFnvP;
      } else {
        h = (h ^ (w & 0xffu)) * kFnvP;
        h = (h ^ ((w >> 8) & 0xffu)) * kFnvP;
        h = (h ^ ((w >> 16) & 0xffu)) * kFnvP;
        h = (h ^ (w >> 24)) * kFnvP;
        h *= P4;
      }
    }
    __syncthreads();
  }
  if (s < nsub) {
    const unsigned long long a = fnv_pow(kFnvP, 8ull * cnt);
    A[s] = a;
    D[s] = h - a * h_in;
  }
}

// Affine maps h -> A h + D composed in row order, 256 per block:
// (A1, D1) then (A2, D2) = (A2 A1, A2 D1 + D2).
static __global__ void __launch_bounds__(256) fnv_affine_reduce(const unsigned long long* A, const unsigned long long* D,
                                                         uint32_t n, unsigned long long* Ao, unsigned long long* Do) {
  __shared__ unsigned long long sA[256], sD[256];
  const uint32_t i = blockIdx.x * 256u + threadIdx.x;
  sA[threadIdx.x] = i < n ? A[i] : 1ull;
  sD[threadIdx.x] = i < n ? D[i] : 0ull;
  __syncthreads();
  for (uint32_t s = 1; s < 256; s <<= 1) {
    unsigned long long a = 0, d = 0;
    const bool act = (threadIdx.x % (2 * s)) == 0;
    if (act) {
      a = sA[threadIdx.x + s] * sA[threadIdx.x];
      d = sA[threadIdx.x + s] * sD[threadIdx.x] + sD[threadIdx.x + s];
    }
    __syncthreads();
    if (act) {
      sA[threadIdx.x] = a;
      sD[threadIdx.x] = d;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    Ao[blockIdx.x] = sA[0];
    Do[blockIdx.x] = sD[0];
  }
}

static __global__ void fnv_affine_apply(const unsigned long long* A, const unsigned long long* D, unsigned long long* hash) {
  *hash = A[0] * *hash + D[0];
}

}  // namespace nb200
