// FP32 CUDA-core throughput probe: the roofline denominator for the SIMT conv
// (MEASURED_PEAKS.json carries only HBM and bf16 tensor peaks).  EXACT issues
// the conv's own instruction pair (FMUL+FADD, 1 flop/lane/clk); otherwise FFMA.
#include <cuda_runtime.h>
#include <stdint.h>

namespace im2win {

template <bool EXACT>
__global__ void __launch_bounds__(256) fp32_peak_kernel(float* sink, float a, float b, int iters) {
  constexpr int C = 32;
  float acc[C];
#pragma unroll
  for (int j = 0; j < C; ++j) acc[j] = threadIdx.x * 1e-7f + j;
  float bb[C];
#pragma unroll
  for (int j = 0; j < C; ++j) bb[j] = b + j * 1e-6f;
  // each product depends on the running value, so nothing can be hoisted
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < C; ++j) {
      if constexpr (EXACT) acc[j] = __fadd_rn(__fmul_rn(acc[j], a), bb[j]);
      else acc[j] = __fmaf_rn(acc[j], a, bb[j]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < C; ++j) s += acc[j];
  if (s == 1234.5f) sink[threadIdx.x] = s;
}

}  // namespace im2win

extern "C" int im2win_bench_fp32_peak(float* sink, int32_t exact, int32_t iters, int32_t blocks,
                                      void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (exact)
    im2win::fp32_peak_kernel<true><<<blocks, 256, 0, st>>>(sink, 0.999f, 1.0001f, iters);
  else
    im2win::fp32_peak_kernel<false><<<blocks, 256, 0, st>>>(sink, 0.999f, 1.0001f, iters);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
