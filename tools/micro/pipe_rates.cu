// Issue rates of the instructions the temporal-blocked step kernel is built
// from (B200, sm_100a), to decide which pipe each part of the car update
// should use.  Every kernel runs 8 independent dependency chains per
// thread, 16 warps per SM (4 per SMSP), on every SM; prints warp
// instructions per SMSP cycle (clock64 around the loop).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_rates tools/micro/pipe_rates.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kIter = 2048;

template <int K>
__device__ __forceinline__ void op(uint32_t& a, uint32_t p, uint32_t q) {
  if constexpr (K == 0) asm volatile("max.s32 %0, %0, %1;" : "+r"(a) : "r"(p));                 // VIMNMX
  if constexpr (K == 1) asm volatile("{.reg .u32 t; add.u32 t, %0, %1; min.u32 %0, t, %2;}" : "+r"(a) : "r"(p), "r"(q));  // VIADDMNMX
  if constexpr (K == 2) asm volatile("{.reg .f32 t; mov.b32 t, %0; min.f32 t, t, %1, %2; mov.b32 %0, t;}" : "+r"(a) : "f"(__uint_as_float(p)), "f"(__uint_as_float(q)));  // FMNMX3
  if constexpr (K == 3) asm volatile("{.reg .s32 t; shr.s32 t, %1, 31; add.s32 %0, %0, t;}" : "+r"(a) : "r"(a ^ p));  // LEA.HI.SX32-ish
  if constexpr (K == 4) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(p), "r"(q));    // IMAD
  if constexpr (K == 5) asm volatile("{.reg .u64 w; mul.wide.u32 w, %0, %1; cvt.u32.u64 %0, w;}" : "+r"(a) : "r"(p));  // IMAD.WIDE
  if constexpr (K == 6) asm volatile("{.reg .f32 t; mov.b32 t, %0; add.rn.f32 t, t, %1; mov.b32 %0, t;}" : "+r"(a) : "f"(__uint_as_float(p)));  // FADD reg
  if constexpr (K == 7) asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(a) : "r"(p), "r"(q));  // IADD3
  if constexpr (K == 8) asm volatile("{.reg .f32 t; mov.b32 t, %0; add.rn.f32 t, t, 0f00000001; mov.b32 %0, t;}" : "+r"(a));  // FADD imm
  if constexpr (K == 9) asm volatile("{.reg .u32 t; add.u32 t, %0, %1; max.u32 %0, t, %2;}" : "+r"(a) : "r"(p), "r"(q));  // VIADDMNMX max
  if constexpr (K == 10) asm volatile("{.reg .u32 lo, hi; .reg .u64 w; mul.wide.u32 w, %0, %1; mov.b64 {lo, hi}, w; shr.u32 lo, lo, 1; add.u32 %0, lo, hi;}" : "+r"(a) : "r"(p));  // IMAD.WIDE + LEA.HI
}

template <int K>
__global__ void __launch_bounds__(128) kern(uint32_t* out, uint32_t p, uint32_t q, unsigned long long* cyc) {
  uint32_t a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = threadIdx.x * 7u + c + blockIdx.x;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < kIter; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) op<K>(a[c], p + c, q);
  }
  __syncthreads();
  const long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) atomicMax(cyc, static_cast<unsigned long long>(t1 - t0));
}

template <int K>
void run(const char* name, int sms, uint32_t* out, unsigned long long* cyc) {
  cudaMemset(cyc, 0, 8);
  kern<K><<<sms * 4, 128>>>(out, 3u, 0x7fffffffu, cyc);  // 4 blocks x 4 warps = 16 warps per SM
  kern<K><<<sms * 4, 128>>>(out, 3u, 0x7fffffffu, cyc);
  cudaDeviceSynchronize();
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  // per SMSP: 4 warps x kIter x 8 warp-instructions (per op) in c cycles
  const double per = 4.0 * kIter * 8 / static_cast<double>(c);
  printf("{\"op\": \"%s\", \"warp_ops_per_smsp_cycle\": %.3f}\n", name, per);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out;
  unsigned long long* cyc;
  cudaMalloc(&out, sms * 4 * 128 * 4);
  cudaMalloc(&cyc, 8);
  run<0>("VIMNMX max.s32", sms, out, cyc);
  run<1>("VIADDMNMX add+min.u32", sms, out, cyc);
  run<2>("FMNMX3 min.f32 x3", sms, out, cyc);
  run<3>("shr.s32+add (LEA.HI.SX32)", sms, out, cyc);
  run<4>("IMAD mad.lo.u32", sms, out, cyc);
  run<5>("IMAD.WIDE mul.wide.u32", sms, out, cyc);
  run<6>("FADD reg", sms, out, cyc);
  run<7>("IADD3 add+add", sms, out, cyc);
  run<8>("FADD imm", sms, out, cyc);
  run<9>("VIADDMNMX add+max.u32", sms, out, cyc);
  run<10>("IMAD.WIDE+LEA.HI (per pair)", sms, out, cyc);
  return 0;
}
