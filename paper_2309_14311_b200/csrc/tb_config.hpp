// tb_config.hpp -- geometry of the temporal-blocked step kernel, shared by
// the single-GPU engine (engine.cu) and the segmented ring (sharded.cu).
#pragma once
#include <cstdint>

#include "minstd.hpp"  // NB_HD

namespace nb200 {

// Measured on C3 (tools/variants, round 1): 128 threads x 16 cars with
// __launch_bounds__(128, 5) (95 registers, 20 warps/SM) beat 256x8 by 13 %
// and 128x16 unconstrained (140 registers) by 8 %.
#ifndef NB_TB_TPB
#define NB_TB_TPB 128
#endif
#ifndef NB_TB_CPT
#define NB_TB_CPT 32
#endif
#ifndef NB_TB_MINB
#define NB_TB_MINB 4
#endif
// Halo depth = the deepest temporal blocking a launch may use (k <= HALO).
#ifndef NB_TB_HALO
#define NB_TB_HALO 32
#endif

#ifndef NB_TB_WT
#define NB_TB_WT 1
#endif

// Per-step velocity sum of a thread's cars: 0 IADD3 (ALU pipe), 1 FP32
// denormal adds (FMA pipe, step_kernels.cuh vsum_fp32), 2 IMAD tree.
// Measured on C3 (round 2, tools/variant_bench.py): 0 2.14e12, 1 2.18e12,
// 2 2.06e12 (with NB_TB_MN3); half IADD3 / half FP32 2.11e12.
#ifndef NB_TB_VSUM
#define NB_TB_VSUM 1
#endif
// Velocity clamp min(v + 1, vmax, gap) as one FMNMX3 (tb_kernel.cuh).
#ifndef NB_TB_MN3
#define NB_TB_MN3 1
#endif

// L2 bulk prefetch of each warp's next tile (tb_kernel.cuh).
// 1: a warp tile whose cars all take the plain path keeps its positions
// relative to the warp's first car (< 2^24, so FP32 adds on the bit patterns
// are exact): the headway and the move become FADDs on the FP32 lanes instead
// of two IMADs on the FMA-heavy pipe.  Bit-exact (parity suite green), but
// measured 0.7 % SLOWER on C3 and C5 (2.156e12 vs 2.171e12, 2.074e12 vs
// 2.091e12; tools/ab_libs.py, round 2): the FMA-heavy pipe is not what holds
// the kernel back.  Off.
#ifndef NB_TB_FREL
#define NB_TB_FREL 0
#endif
#ifndef NB_TB_PREFETCH
#define NB_TB_PREFETCH 0
#endif

// Tile geometry.  Block tiles (WT = false): the block's TPB*CPT cars share
// one 16-car halo and hand leaders across warps through shared memory (one
// barrier per step).  Warp tiles (WT = true): each warp owns 32*CPT - 16
// cars with its own halo and never synchronises with the other warps.
template <int TPB, int CPT, int HALO, bool WT>
struct TbGeom {
  static constexpr uint32_t kWarpLoad = WT ? 32u * CPT : uint32_t(TPB) * CPT;  // one halo per ...
  static constexpr uint32_t kWarpStore = kWarpLoad - HALO;                     // ... this many owned
  static constexpr uint32_t kStore = WT ? (TPB / 32) * kWarpStore : kWarpStore;  // owned per block tile
  static constexpr uint32_t kLoad = kStore + HALO;                              // block tile's extent
  // First car of thread t within its block tile.
  static constexpr NB_HD uint32_t offset(uint32_t t) {
    return WT ? (t / 32) * kWarpStore + (t % 32) * CPT : t * CPT;
  }
};

// Grid of the temporal-blocked kernels: kTbWaves times the resident blocks
// (148 SMs x 5), so the hardware hands tiles out in ~10 block waves.  A
// persistent grid (one wave, static grid-stride tiles) finishes when its
// slowest SM does: on C3 one wave measured 1.63e12 car-updates/s, 2 waves
// 1.68e12, 4 1.73e12, 10 1.75e12, 40 1.72e12, one tile per block 1.65e12
// (round 1, tools/grid_sweep.py).  Env NASCH_B200_WAVES overrides.
#ifndef NB_TB_WAVES
#define NB_TB_WAVES 10
#endif
constexpr int kTbWaves = NB_TB_WAVES;

constexpr int kTbTPB = NB_TB_TPB;                   // threads per tile
constexpr int kTbCPT = NB_TB_CPT;                   // consecutive cars per thread
constexpr int kTbHalo = NB_TB_HALO;                 // cars ahead re-read per tile (>= K)
constexpr bool kTbWT = NB_TB_WT != 0;
using TbLarge = TbGeom<kTbTPB, kTbCPT, kTbHalo, kTbWT>;
constexpr uint32_t kTbLoad = TbLarge::kLoad;        // cars spanned per tile
constexpr uint32_t kTbStore = TbLarge::kStore;      // cars owned per tile

// Medium rings: narrower tiles so every SM gets work.
constexpr int kTbmTPB = 128;
constexpr int kTbmCPT = 4;
using TbMedium = TbGeom<kTbmTPB, kTbmCPT, kTbHalo, false>;
constexpr uint32_t kTbmLoad = TbMedium::kLoad;      // 512
constexpr uint32_t kTbmStore = TbMedium::kStore;    // 496

}  // namespace nb200
