// minstd.hpp -- counter-based restatement of the reference's single
// shared minstd stream (a = 48271, c = 0, m = 2^31-1; src/lcg.hpp:21-56).
//
// The reference draws the (t*N + r + 1)-th generator output for the car of
// rank r at step t (one draw per car per step in rank order,
// src/model.cpp:42-75, src/engine.cpp:62-72 + 115-145).  With c = 0 and m
// prime that output is s0 * a^(t*N + r + 1) mod m, with exponents reducible
// mod (m-1) (Fermat), so any draw is O(1) mulmods away from any other --
// this is what makes the GPU step independent of launch geometry and GPU
// count, as the reference's jump-ahead does for OpenMP team size.
//
// The Bernoulli test `double(s)/double(m) < p` (src/model.cpp:51) is
// replaced by the exact integer test `s < threshold(p)`: IEEE division is
// correctly rounded hence monotone in s, so {s : fl(s/m) < p} is a prefix
// [0, T_p) of the integers, and T_p is found by bisection with the very
// same binary64 expression (tests/test_capi_host.py test_threshold_* check
// the boundary).
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define NB_HD __host__ __device__ __forceinline__
#else
#define NB_HD inline
#endif

namespace nb200 {

constexpr uint32_t kA = 48271u;         // src/lcg.hpp:22
constexpr uint32_t kM = 2147483647u;    // src/lcg.hpp:23
constexpr uint64_t kOrder = kM - 1ull;  // multiplicative order bound

// x*y mod (2^31-1) for x, y < 2^31: Mersenne fold of the <2^62 product.
NB_HD uint32_t mulmod(uint32_t x, uint32_t y) {
  const uint64_t p = static_cast<uint64_t>(x) * y;
  uint32_t r = static_cast<uint32_t>(p & kM) + static_cast<uint32_t>(p >> 31);
  return r >= kM ? r - kM : r;
}

#if defined(__CUDACC__)
// Device hot-path form: the final conditional subtract as an unsigned min
// (r - m wraps above r unless r >= m), which ptxas fuses into VIADDMNMX.
__device__ __forceinline__ uint32_t mulmod_d(uint32_t x, uint32_t y) {
  const uint64_t p = static_cast<uint64_t>(x) * y;
  const uint32_t r = static_cast<uint32_t>(p & kM) + static_cast<uint32_t>(p >> 31);
  return min(r, r - kM);
}

// Same product with the multiplier given doubled (x2 = 2x < 2^32): the fold
// term p >> 31 is then the high word of x2*y.  The product is one 64-bit
// IMAD.WIDE.U32 (FMA pipe) and hi + (lo >> 1) one LEA.HI (ALU pipe);
// separate mul.lo/mul.hi let ptxas fold the shift into IMAD.HI's 64-bit
// addend, which needs a zeroed register per car (an extra IMAD.MOV/HFMA2):
// measured +6 % on C3/C5/C4 for the wide form (round 1,
// tools/variant_bench.py).
__device__ __forceinline__ uint32_t mulmod_x2(uint32_t x2, uint32_t y) {
  uint32_t lo, hi;
  asm("{ .reg .u64 p; mul.wide.u32 p, %2, %3; mov.b64 {%0, %1}, p; }" : "=r"(lo), "=r"(hi) : "r"(x2), "r"(y));
  // x2*y = 2p: lo holds bits 1..31 of p shifted up one; p & m = lo >> 1
  const uint32_t r = (lo >> 1) + hi;
  return min(r, r - kM);
}
#endif

// a^e mod m by square-and-multiply (host side / one-off device use).
NB_HD uint32_t powmod(uint32_t base, uint64_t e) {
  e %= kOrder;
  uint32_t result = 1, b = base % kM;
  while (e) {
    if (e & 1) result = mulmod(result, b);
    b = mulmod(b, b);
    e >>= 1;
  }
  return result;
}

// src/lcg.cpp:11-16: state = seed mod m, zero escapes to one.
NB_HD uint32_t seeded(uint64_t seed) {
  const uint32_t s = static_cast<uint32_t>(seed % kM);
  return s == 0 ? 1u : s;
}

// Exponent (t*N + 1 + w) mod (m-1) without overflow; t, n arbitrary u64.
NB_HD uint64_t draw_exponent(uint64_t t, uint64_t n, uint64_t w) {
  const uint64_t tn = ((t % kOrder) * (n % kOrder)) % kOrder;
  return (tn + 1 + (w % kOrder)) % kOrder;
}

// Compile-time power tables: lin[i] = a^i (i < 256), sq[b] = a^(2^b).
struct PowTables {
  uint32_t lin[256];
  uint32_t sq[32];
};
constexpr uint32_t cx_mulmod(uint32_t x, uint32_t y) {
  const uint64_t p = static_cast<uint64_t>(x) * y;
  const uint32_t r = static_cast<uint32_t>(p & kM) + static_cast<uint32_t>(p >> 31);
  return r >= kM ? r - kM : r;
}
constexpr PowTables make_pow_tables() {
  PowTables t{};
  t.lin[0] = 1;
  for (int i = 1; i < 256; ++i) t.lin[i] = cx_mulmod(t.lin[i - 1], kA);
  t.sq[0] = kA;
  for (int b = 1; b < 32; ++b) t.sq[b] = cx_mulmod(t.sq[b - 1], t.sq[b - 1]);
  return t;
}

// Doubled powers 2 a^c (c < 64): the per-car draw multipliers of the
// temporal-blocked kernel, read as constant-bank operands of IMAD.WIDE.
struct Pow2Table {
  uint32_t v[64];
};
constexpr Pow2Table make_pow2_table() {
  Pow2Table t{};
  uint32_t a = 1;
  for (int i = 0; i < 64; ++i) {
    t.v[i] = a << 1;
    a = cx_mulmod(a, kA);
  }
  return t;
}

#if defined(__CUDACC__)
static __constant__ PowTables c_pow = make_pow_tables();
static __constant__ Pow2Table c_apow2 = make_pow2_table();

// a^e mod m computed by a whole warp (every lane calls it with the same e;
// every lane gets the result): lane b contributes a^(2^b) if bit b of the
// reduced exponent is set, then a 5-level butterfly of mulmods.  ~40
// cycles of latency instead of the ~31 dependent squarings of powmod.
__device__ __forceinline__ uint32_t powmod_warp(uint64_t e) {
  const uint32_t er = static_cast<uint32_t>(e % kOrder);  // < 2^31
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t r = (lane < 31 && ((er >> lane) & 1u)) ? c_pow.sq[lane] : 1u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r = mulmod_d(r, __shfl_xor_sync(0xffffffffu, r, o));
  return r;
}
#endif

// Host-only: smallest s in [0, m] with double(s)/double(m) >= p.
inline uint32_t deceleration_threshold(double p) {
  uint64_t lo = 0, hi = kM;  // invariant: answer in [lo, hi]
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (static_cast<double>(mid) / static_cast<double>(kM) < p) {
      lo = mid + 1;
    } else {
      hi = mid;
    }
  }
  return static_cast<uint32_t>(lo);
}

}  // namespace nb200
