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


// ---- nibble decomposition of the row digest (GpuRing) ---------------------
//
// The 256-start tables above do the 64-bit FNV work 256 times over.  One byte
// maps h -> (h xor b) * P, and bit k of the result depends only on bits <= k
// of h (P is odd, xor is bitwise).  So the low nibble evolves on its own,
//     l -> ((l xor b) * P) mod 16            (P mod 16 = 3),
// the low byte on its own once its low nibble is known, and once the low
// byte is known at every point a run of bytes maps h -> P^(8n) h + d, which
// is affine.  A step's digest is therefore computed in three passes over the
// row, each far cheaper than tracking all 256 low bytes:
//   A  fnv_nib_kernel<VT, 0>  one LANE per chunk (4 slots of 512 values):
//                             the chunk's low-nibble map for starts 0..7,
//                             four per register in 8-bit lanes (one LOP3 +
//                             one IMAD per byte and register); flipping bit 3
//                             commutes with both operations, F(l ^ 8) =
//                             F(l) ^ 8, which gives starts 8..15;
//      fnv_up16 / fnv_down16  the chunk maps composed 256 at a time up a tree
//                             (each map's prefix table kept), then every
//                             chunk's true incoming low nibble gathered down
//                             it from the running digest's;
//   B  fnv_nib_kernel<VT, 1>  one lane per chunk, from its true low nibble:
//                             the high nibble's map for starts 0..7 (bit 7
//                             commutes), two per register in 16-bit lanes,
//                             and the full byte at each slot boundary;
//                             composed the same way -> every chunk's true
//                             incoming low byte;
//   C  fnv_exact_kernel       one lane per slot, the exact 64-bit FNV of its
//                             values from its true low byte: the slot maps
//                             the true state h to P^(8n) h + d; the slots'
//                             maps reduced in row order (fnv_affine_reduce)
//                             and applied to the digest.
// Slots are ID-aligned, so a lane streams its values with 16-byte loads.  The
// row (rank r = id (head + r) mod N) starts inside unit head / 512, which is
// split in two: [head, end of that unit), the following units in id order
// (wrapping), then [unit start, head).  Every array has nu + 1 slots (the
// last one empty when head is unit-aligned), so the geometry -- and the
// captured graph -- is the same every step.
constexpr uint32_t kFnvSlot = 512;          // row values per slot (ID-aligned)
constexpr uint32_t kFnvSlotsPerChunk = 4;   // slots per pass A/B lane
constexpr uint32_t kFnvP8 = 0xb3u;          // P mod 256
constexpr uint32_t kFnvP8_5 = (kFnvP8 * kFnvP8 * kFnvP8 * kFnvP8 * kFnvP8) & 0xffu;  // last data byte + 4 zero bytes
constexpr uint32_t kFnvP8_8 = (kFnvP8_5 * kFnvP8 * kFnvP8 * kFnvP8) & 0xffu;       // u8 value: 1 byte + 7 zero bytes
constexpr uint32_t kFnvP4 = kFnvP8 & 0xfu;      // P mod 16 (= 3)
constexpr uint32_t kFnvP4_5 = kFnvP8_5 & 0xfu;  // (= 3)
constexpr uint32_t kFnvP4_8 = kFnvP8_8 & 0xfu;  // (= 1)

__host__ __device__ constexpr unsigned long long fnv_pow_c(uint64_t e) {
  unsigned long long r = 1, b = kFnvP;
  while (e) {
    if (e & 1) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}
constexpr unsigned long long kFnvPSlot = fnv_pow_c(8ull * kFnvSlot);  // P^(8 * 512): a full slot's slope

struct FnvRow {
  uint32_t N, head, nu, hu;  // cars, head id, units per array, head unit
  uint32_t npos;             // slots per array: nu + 1, rounded up to whole chunks (the rest empty)
  uint32_t pos_only;         // no velocity part: its slots are empty
};

__device__ __forceinline__ FnvRow fnv_row(uint32_t N, uint32_t W, uint32_t pos_only = 0) {
  FnvRow r;
  r.pos_only = pos_only;
  r.N = N;
  r.head = (N - W) % N;
  r.nu = (N + kFnvSlot - 1) / kFnvSlot;
  r.hu = r.head / kFnvSlot;
  r.npos = (r.nu + 1 + kFnvSlotsPerChunk - 1) / kFnvSlotsPerChunk * kFnvSlotsPerChunk;
  return r;
}

// Slot s of the row: array (0 positions, 1 velocities) and id range [a, b).
__device__ __forceinline__ void fnv_slot(const FnvRow& r, uint32_t s, uint32_t& arr, uint32_t& a, uint32_t& b) {
  arr = s >= r.npos ? 1u : 0u;
  const uint32_t t = arr ? s - r.npos : s;
  if (arr && r.pos_only) {
    a = b = 0;
  } else if (t == 0) {
    a = r.head;
    b = min(r.hu * kFnvSlot + kFnvSlot, r.N);
  } else if (t >= r.nu) {
    a = t == r.nu ? r.hu * kFnvSlot : 0u;
    b = t == r.nu ? r.head : 0u;
  } else {
    uint32_t u = r.hu + t;
    if (u >= r.nu) u -= r.nu;
    a = u * kFnvSlot;
    b = min(a + kFnvSlot, r.N);
  }
}

// Per-warp staging of the lanes' slots: every lane streams its own slot, so
// direct per-lane loads would touch 32 cache lines per instruction.  Instead
// the warp copies 256-byte windows of all 32 slots into shared memory with
// coalesced 16-byte cp.async copies (a row = one lane's window; rows padded
// by 16 bytes, so the lanes' 16-byte reads of their own rows hit distinct
// bank groups), then each lane reads its row.
constexpr uint32_t kFnvWin = 256;  // bytes per row and window
struct FnvStage {
  uint4 tile[32][kFnvWin / 16 + 1];
  const char* base[32];
  uint32_t bytes[32];
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Visits the values of ids [a, b) of one array in order: f4(w) for a 4-byte
// value (positions; u32 velocities), f1(w, k) for byte k of w holding a u8
// velocity.  Warp-collective (every lane calls it; an idle lane passes an
// empty range): full slots (ID-aligned, 512 values) go through the staged
// windows, the few partial ones (the split head slot, the short last unit)
// value by value afterwards.
template <typename VT, typename F4, typename F1>
__device__ __forceinline__ void fnv_slot_values(FnvStage& st, const uint32_t* X, const VT* V, uint32_t arr,
                                                uint32_t a, uint32_t b, F4&& f4, F1&& f1) {
  const uint32_t lane = threadIdx.x & 31u;
  const bool full = b - a == kFnvSlot;
  const bool wide = arr == 0 || sizeof(VT) == 4;
  const uint32_t bytes = full ? kFnvSlot * (wide ? 4u : 1u) : 0u;
  st.base[lane] = wide ? reinterpret_cast<const char*>((arr == 0 ? X : reinterpret_cast<const uint32_t*>(V)) + a)
                       : reinterpret_cast<const char*>(V) + a;
  st.bytes[lane] = bytes;
  __syncwarp();
  const uint32_t most = __reduce_max_sync(0xffffffffu, bytes);
  for (uint32_t w = 0; w < most; w += kFnvWin) {
#pragma unroll
    for (uint32_t it = 0; it < 32 * (kFnvWin / 16) / 32; ++it) {
      const uint32_t idx = it * 32 + lane;
      const uint32_t r = idx / (kFnvWin / 16), u = idx % (kFnvWin / 16);
      if (w < st.bytes[r]) cp_async16(&st.tile[r][u], st.base[r] + w + 16 * u);
    }
    cp_async_wait_all();
    __syncwarp();
    if (w < bytes) {
      // partial unrolling: the fully unrolled window (2.3k instructions per
      // lane in pass B) missed the instruction cache
      if (wide) {
#pragma unroll 4
        for (uint32_t u = 0; u < kFnvWin / 16; ++u) {
          const uint4 q = st.tile[lane][u];
          f4(q.x);
          f4(q.y);
          f4(q.z);
          f4(q.w);
        }
      } else {
#pragma unroll 2
        for (uint32_t u = 0; u < kFnvWin / 16; ++u) {
          const uint4 q = st.tile[lane][u];
          f1(q.x, 0); f1(q.x, 1); f1(q.x, 2); f1(q.x, 3);
          f1(q.y, 0); f1(q.y, 1); f1(q.y, 2); f1(q.y, 3);
          f1(q.z, 0); f1(q.z, 1); f1(q.z, 2); f1(q.z, 3);
          f1(q.w, 0); f1(q.w, 1); f1(q.w, 2); f1(q.w, 3);
        }
      }
    }
    __syncwarp();
  }
  if (!full) {
    for (uint32_t id = a; id < b; ++id) {
      if (arr == 0) f4(__ldg(X + id));
      else if (sizeof(VT) == 4) f4(static_cast<uint32_t>(__ldg(V + id)));
      else f1(static_cast<uint32_t>(__ldg(V + id)), 0);
    }
  }
}

// Byte k of w broadcast to the four 8-bit lanes / the two 16-bit lanes.
__device__ __forceinline__ uint32_t fnv_bcast8(uint32_t w, int k) { return __byte_perm(w, 0u, 0x1111u * k); }
__device__ __forceinline__ uint32_t fnv_bcast16(uint32_t w, int k) { return __byte_perm(w, 0u, 0x4040u | (0x0101u * k)); }

// Passes A (LEVEL 0) and B (LEVEL 1) of chunk c (slots 4c .. 4c+3).
// Out: F[c][16] (A: low nibble out per low nibble in; B: high nibble out per
// high nibble in); B also Fsub[c][q][16], the full byte after slot q < 3 per
// high nibble in.  Warp-collective (the staging); `live` false: no output.
template <typename VT, int LEVEL>
__device__ __forceinline__ void fnv_nib_chunk(FnvStage& st, const FnvRow& row, const uint32_t* X, const VT* V,
                                              uint32_t c, bool live, const uint8_t* lo4, uint8_t* F,
                                              uint8_t* Fsub) {
  const uint32_t nslots = 2 * row.npos;
  const uint32_t s0 = c * kFnvSlotsPerChunk;
  uint32_t out[16];
  if (LEVEL == 0) {
    constexpr uint32_t M = 0x0f0f0f0fu;
    uint32_t h0 = 0x03020100u, h1 = 0x07060504u;  // starts 0..3, 4..7
    auto f4 = [&](uint32_t w) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t bb = fnv_bcast8(w, k);
        const uint32_t mul = k < 3 ? kFnvP4 : kFnvP4_5;
        h0 = ((h0 ^ bb) & M) * mul;
        h1 = ((h1 ^ bb) & M) * mul;
      }
    };
    auto f1 = [&](uint32_t w, int k) {
      const uint32_t bb = fnv_bcast8(w, k);
      h0 = ((h0 ^ bb) & M) * kFnvP4_8;
      h1 = ((h1 ^ bb) & M) * kFnvP4_8;
    };
    for (uint32_t q = 0; q < kFnvSlotsPerChunk; ++q) {
      uint32_t arr = 0, a = 0, b = 0;
      if (live && s0 + q < nslots) fnv_slot(row, s0 + q, arr, a, b);
      fnv_slot_values<VT>(st, X, V, arr, a, b, f4, f1);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      out[j] = (h0 >> (8 * j)) & 0xfu;
      out[j + 4] = (h1 >> (8 * j)) & 0xfu;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) out[j + 8] = out[j] ^ 8u;
  } else {
    constexpr uint32_t M = 0x00ff00ffu;
    const uint32_t lo = live ? lo4[c] : 0u;
    // register i: start i in the low half, start i + 4 in the high half
    uint32_t g[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) g[i] = ((uint32_t(i) << 4) | lo) | ((((uint32_t(i) + 4u) << 4) | lo) << 16);
    auto f4 = [&](uint32_t w) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t bb = fnv_bcast16(w, k);
        const uint32_t mul = k < 3 ? kFnvP8 : kFnvP8_5;
#pragma unroll
        for (int i = 0; i < 4; ++i) g[i] = ((g[i] ^ bb) & M) * mul;
      }
    };
    auto f1 = [&](uint32_t w, int k) {
      const uint32_t bb = fnv_bcast16(w, k);
#pragma unroll
      for (int i = 0; i < 4; ++i) g[i] = ((g[i] ^ bb) & M) * kFnvP8_8;
    };
    auto byte_of = [&](int j) { return (g[j & 3] >> (16 * (j >> 2))) & 0xffu; };
    for (uint32_t q = 0; q < kFnvSlotsPerChunk; ++q) {
      uint32_t arr = 0, a = 0, b = 0;
      if (live && s0 + q < nslots) fnv_slot(row, s0 + q, arr, a, b);
      fnv_slot_values<VT>(st, X, V, arr, a, b, f4, f1);
      if (live && q + 1 < kFnvSlotsPerChunk) {
        uint8_t* sub = Fsub + (size_t(c) * (kFnvSlotsPerChunk - 1) + q) * 16;
        uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t y = byte_of(j);
          w[j >> 2] |= y << (8 * (j & 3));
          w[(j + 8) >> 2] |= (y ^ 0x80u) << (8 * (j & 3));
        }
        *reinterpret_cast<uint4*>(sub) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      out[j] = byte_of(j) >> 4;
      out[j + 8] = out[j] ^ 8u;
    }
  }
  if (!live) return;
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    w[i] = out[4 * i] | (out[4 * i + 1] << 8) | (out[4 * i + 2] << 16) | (out[4 * i + 3] << 24);
  *reinterpret_cast<uint4*>(F + size_t(c) * 16) = make_uint4(w[0], w[1], w[2], w[3]);
}

// Lane = chunk c.  (Pairing a position chunk with a velocity chunk per lane
// evens the warps' work but halves the warps: measured slower.)
constexpr uint32_t kFnvTPB = 128;  // 4 warps: 4 x 9 KB staging
template <typename VT, int LEVEL>
__global__ void __launch_bounds__(kFnvTPB) fnv_nib_kernel(const RingArgs ra, const uint8_t* lo4, uint8_t* F,
                                                          uint8_t* Fsub) {
  __shared__ FnvStage stage[kFnvTPB / 32];
  FnvStage& st = stage[threadIdx.x / 32];
  const Ctl* ctl = ra.ctl;
  const FnvRow row = fnv_row(ra.n, ctl->W, ra.fnv_pos_only);
  const uint32_t nchunks = 2 * row.npos / kFnvSlotsPerChunk;
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if ((c & ~31u) >= nchunks) return;  // whole warps only: the staging is warp-collective
  const int bsel = static_cast<int>(ctl->buf);
  const uint32_t* X = xbuf(ra, bsel);
  const VT* V = vbuf<VT>(ra, bsel);
  fnv_nib_chunk<VT, LEVEL>(st, row, X, V, c, c < nchunks, lo4, F, Fsub);
}

// Composition tree over maps of 16 nibbles: block = kUpGroups groups of 256
// maps, thread = (group, start l) following l through its group's maps
// (staged in shared memory, rows padded so the groups use distinct banks);
// records pre[m][l], the value entering map m from start l of m's group, and
// the group's composed map out[g].
constexpr uint32_t kUpGroups = 8;
static __global__ void __launch_bounds__(16 * kUpGroups) fnv_up16_kernel(const uint8_t* maps, uint32_t n, uint8_t* pre,
                                                                        uint8_t* out) {
  __shared__ uint4 s[kUpGroups][257];
  const uint32_t g0 = blockIdx.x * kUpGroups;
  const uint4* src = reinterpret_cast<const uint4*>(maps);
  for (uint32_t i = threadIdx.x; i < kUpGroups * 256; i += blockDim.x) {
    const uint32_t m = g0 * 256 + i;
    s[i / 256][i % 256] = m < n ? src[m] : make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  const uint32_t gl = threadIdx.x / 16, l = threadIdx.x % 16;
  const uint32_t g = g0 + gl;
  if (size_t(g) * 256 >= n) return;
  const uint32_t cnt = min(256u, n - g * 256);
  const uint8_t* sm = reinterpret_cast<const uint8_t*>(&s[gl][0]);
  uint8_t* pg = pre + size_t(g) * 256 * 16 + l;
  uint32_t v = l;
  for (uint32_t i = 0; i < cnt; ++i) {
    pg[i * 16] = static_cast<uint8_t>(v);
    v = sm[i * 16 + v];
  }
  out[size_t(g) * 16 + l] = static_cast<uint8_t>(v);
}

// Down the tree: lb[m] = pre[m][up[m / 256]], the value entering map m; at
// the top the value entering the row is the digest's nibble (hash >> shift).
static __global__ void __launch_bounds__(256) fnv_down16_kernel(const uint8_t* pre, uint32_t n, const uint8_t* up,
                                                               const unsigned long long* hash, int shift,
                                                               uint8_t* lb) {
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  const uint32_t u = up ? up[m / 256] : static_cast<uint32_t>((*hash >> shift) & 0xfu);
  lb[m] = pre[size_t(m) * 16 + u];
}

// Pass C: one slot, from its true incoming low byte (chunk start: low and
// high nibble from passes A and B; later slots: pass B's boundary bytes),
// the exact 64-bit FNV of its values: the slot maps the true state h to
// A h + D with A = P^(8n).  Warp-collective.
template <typename VT>
__device__ __forceinline__ void fnv_exact_slot(FnvStage& st, const FnvRow& row, const uint32_t* X, const VT* V,
                                               uint32_t s, bool live, const uint8_t* lo4, const uint8_t* hi4,
                                               const uint8_t* Fsub, unsigned long long* A, unsigned long long* D) {
  const uint32_t c = s / kFnvSlotsPerChunk, q = s % kFnvSlotsPerChunk;
  uint32_t start = 0, arr = 0, a = 0, b = 0;
  if (live) {
    const uint32_t hn = hi4[c];
    start = q == 0 ? (lo4[c] | (hn << 4)) : Fsub[(size_t(c) * (kFnvSlotsPerChunk - 1) + q - 1) * 16 + hn];
    fnv_slot(row, s, arr, a, b);
  }
  unsigned long long h = start;
  constexpr unsigned long long P8 = fnv_pow_c(8);
  fnv_slot_values<VT>(st, X, V, arr, a, b, [&](uint32_t w) { h = fnv_value(h, w); },
                      [&](uint32_t w, int k) { h = (h ^ ((w >> (8 * k)) & 0xffu)) * P8; });
  if (!live) return;
  const unsigned long long an = b - a == kFnvSlot ? kFnvPSlot : fnv_pow(kFnvP, 8ull * (b - a));
  A[s] = an;
  D[s] = h - an * start;
}

// Lane = slot s.
template <typename VT>
__global__ void __launch_bounds__(kFnvTPB) fnv_exact_kernel(const RingArgs ra, const uint8_t* lo4, const uint8_t* hi4,
                                                            const uint8_t* Fsub, unsigned long long* A,
                                                            unsigned long long* D) {
  __shared__ FnvStage stage[kFnvTPB / 32];
  FnvStage& st = stage[threadIdx.x / 32];
  const Ctl* ctl = ra.ctl;
  const FnvRow row = fnv_row(ra.n, ctl->W, ra.fnv_pos_only);
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if ((s & ~31u) >= 2 * row.npos) return;  // whole warps only
  const int bsel = static_cast<int>(ctl->buf);
  const uint32_t* X = xbuf(ra, bsel);
  const VT* V = vbuf<VT>(ra, bsel);
  fnv_exact_slot<VT>(st, row, X, V, s, s < 2 * row.npos, lo4, hi4, Fsub, A, D);
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
