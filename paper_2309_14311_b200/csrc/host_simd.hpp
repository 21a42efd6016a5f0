// host_simd.hpp -- host-side conversions at the C ABI (u64 <-> the engine's
// u32 positions / u8 or u32 velocities).  The rank-ordered u64 arrays of
// nasch_sim_state / nasch_sim_set_state are 3.2 GB each on BASELINE config
// 3, so these loops set the end-to-end time; with AVX-512 the widening
// writes use non-temporal stores (no read-for-ownership of the destination).
#pragma once
#include <cstddef>
#include <cstdint>

namespace nb200 {

// dst[i] = src[i] for i < n.
void widen_u32(const uint32_t* src, uint64_t* dst, size_t n);
void widen_u8(const uint8_t* src, uint64_t* dst, size_t n);

// Narrows rank-ordered u64 input into (x32, v) and validates it exactly as
// the scalar rules of load_state: returns 0, or the first violated rule
// (1: x >= L, 2: x not increasing, 3: v > vmax, 4: v > vlim) found in
// [lo, hi); `prev` is x[lo - 1] (ignored when lo == 0).
int narrow_validate(const uint64_t* x, const uint64_t* v, size_t lo, size_t hi, uint64_t L, uint64_t vmax,
                    uint64_t vlim, uint32_t* x32, void* vout, int vbytes);

}  // namespace nb200
