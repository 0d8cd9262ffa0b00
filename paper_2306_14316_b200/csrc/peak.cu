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

// The conv's packed form of the exact pair (conv_simt.cu mac_row): rn(a*b) = fma(a, b, -0) and
// rn(c + p) = fma(c, 1, p) on float2 (FFMA2), -0 and 1 opaque kernel arguments; 64 chains.
__global__ void __launch_bounds__(256) fp32_peak_packed_kernel(float* sink, float a, float b, float nz, float one,
                                                              int iters) {
  constexpr int C = 64;
  float acc[C];
#pragma unroll
  for (int j = 0; j < C; ++j) acc[j] = threadIdx.x * 1e-7f + j;
  float bb[C];
#pragma unroll
  for (int j = 0; j < C; ++j) bb[j] = b + j * 1e-6f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < C; j += 2) {
      uint64_t p, c;
      asm("{\n\t.reg .b64 aa, xx, zz;\n\tmov.b64 aa, {%1, %1};\n\tmov.b64 xx, {%2, %3};\n\t"
          "mov.b64 zz, {%4, %4};\n\tfma.rn.f32x2 %0, xx, aa, zz;\n\t}\n"
          : "=l"(p) : "f"(a), "f"(acc[j]), "f"(acc[j + 1]), "f"(nz));
      asm("{\n\t.reg .b64 oo, bbb;\n\tmov.b64 oo, {%2, %2};\n\tmov.b64 bbb, {%3, %4};\n\t"
          "fma.rn.f32x2 %0, %1, oo, bbb;\n\t}\n"
          : "=l"(c) : "l"(p), "f"(one), "f"(bb[j]), "f"(bb[j + 1]));
      asm("mov.b64 {%0, %1}, %2;\n" : "=f"(acc[j]), "=f"(acc[j + 1]) : "l"(c));
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < C; ++j) s += acc[j];
  if (s == 1234.5f) sink[threadIdx.x] = s;
}

}  // namespace im2win

// exact: 0 FFMA chains, 1 FMUL+FADD chains (32 per thread), 2 the packed exact pair (64 per thread)
extern "C" int im2win_bench_fp32_peak(float* sink, int32_t exact, int32_t iters, int32_t blocks,
                                      void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (exact == 2)
    im2win::fp32_peak_packed_kernel<<<blocks, 256, 0, st>>>(sink, 0.999f, 1.0001f, -0.0f, 1.0f, iters);
  else if (exact)
    im2win::fp32_peak_kernel<true><<<blocks, 256, 0, st>>>(sink, 0.999f, 1.0001f, iters);
  else
    im2win::fp32_peak_kernel<false><<<blocks, 256, 0, st>>>(sink, 0.999f, 1.0001f, iters);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
