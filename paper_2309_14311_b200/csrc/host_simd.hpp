// host_simd.hpp -- host-side conversions at the C ABI (u64 <-> the engine's
// u32 positions / u8 or u32 velocities).  The rank-ordered u64 arrays of
// nasch_sim_state / nasch_sim_set_state are 3.2 GB each on BASELINE config
// 3, so these loops set the end-to-end time; with AVX-512 the widening
// writes use non-temporal stores (no read-for-ownership of the destination).
#pragma once
#include <cstddef>
#include <algorithm>
#include <cstdint>
#include <functional>

namespace nb200 {

// dst[i] = src[i] for i < n.
void widen_u32(const uint32_t* src, uint64_t* dst, size_t n);
void widen_u8(const uint8_t* src, uint64_t* dst, size_t n);
// dst[i] = src[i] (u8 velocities into the u32 arrays of nasch_sim_state32).
void widen_u8_u32(const uint8_t* src, uint32_t* dst, size_t n);

// Narrows rank-ordered u64 input into (x32, v) and validates it exactly as
// the scalar rules of load_state: returns 0, or the first violated rule
// (1: x >= L, 2: x not increasing, 3: v > vmax, 4: v > vlim) found in
// [lo, hi); `prev` is x[lo - 1] (ignored when lo == 0).
int narrow_validate(const uint64_t* x, const uint64_t* v, size_t lo, size_t hi, uint64_t L, uint64_t vmax,
                    uint64_t vlim, uint32_t* x32, void* vout, int vbytes);

// The same rules for u32 input (nasch_sim_set_state32, BASELINE's int32
// state); x32 may be null when the positions are uploaded straight from the
// caller's (page-locked) array.
int narrow_validate32(const uint32_t* x, const uint32_t* v, size_t lo, size_t hi, uint64_t L, uint64_t vmax,
                      uint64_t vlim, uint32_t* x32, void* vout, int vbytes);

// Velocities only (set_state32 with page-locked positions, which the device
// validates): narrows v[lo, hi) into vout and returns 4 i + (rule - 1) of the
// first violation (rule 3: v > vmax, 4: v > vlim), or UINT64_MAX.
uint64_t narrow_v32(const uint32_t* v, size_t lo, size_t hi, uint64_t vmax, uint64_t vlim, void* vout, int vbytes);

// Persistent host worker pool (host_simd.cpp): job(i) for i in [0, count)
// on the pool's threads and the caller; returns when all are done.
unsigned host_threads();
void host_run(unsigned count, std::function<void(unsigned)> job);

// Runs f(lo, hi) over [0, n) in parallel host chunks (input validation and
// u64 <-> u32 conversion at the ABI; large rings only).
template <typename F>
void parallel_chunks(size_t n, F&& f) {
  const unsigned nt = static_cast<unsigned>(std::min<size_t>(host_threads(), n / (1u << 20) + 1));
  if (nt <= 1) {
    f(size_t(0), n);
    return;
  }
  const size_t chunk = (n + nt - 1) / nt;
  host_run(nt, [&](unsigned t) {
    const size_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo < hi) f(lo, hi);
  });
}

}  // namespace nb200
