// tb_config.hpp -- geometry of the temporal-blocked step kernel, shared by
// the single-GPU engine (engine.cu) and the segmented ring (sharded.cu).
#pragma once
#include <cstdint>

namespace nb200 {

// Measured on C3 (tools/variants, round 1): 128 threads x 16 cars with
// __launch_bounds__(128, 5) (95 registers, 20 warps/SM) beat 256x8 by 13 %
// and 128x16 unconstrained (140 registers) by 8 %.
#ifndef NB_TB_TPB
#define NB_TB_TPB 128
#endif
#ifndef NB_TB_CPT
#define NB_TB_CPT 16
#endif
#ifndef NB_TB_MINB
#define NB_TB_MINB 5
#endif

constexpr int kTbTPB = NB_TB_TPB;                   // threads per tile
constexpr int kTbCPT = NB_TB_CPT;                   // consecutive cars per thread
constexpr int kTbHalo = 16;                         // cars ahead re-read per tile (>= K)
constexpr uint32_t kTbLoad = kTbTPB * kTbCPT;       // cars loaded per tile
constexpr uint32_t kTbStore = kTbLoad - kTbHalo;    // cars owned per tile

// Medium rings: narrower tiles so every SM gets work.
constexpr int kTbmTPB = 128;
constexpr int kTbmCPT = 4;
constexpr uint32_t kTbmLoad = kTbmTPB * kTbmCPT;    // 512
constexpr uint32_t kTbmStore = kTbmLoad - kTbHalo;  // 496

}  // namespace nb200
