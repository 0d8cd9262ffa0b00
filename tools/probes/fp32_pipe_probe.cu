// FP32 pipe probe (B200): is the packed FFMA2 issue rate the same as FFMA's?
// If so, the bit-exact multiply-then-add (2 roundings) can be issued as
//   p = FFMA2(a, b, -0.0)   == rn(a*b)       (adding -0 is exact, keeps -0)
//   c = FFMA2(c, 1.0, p)    == rn(c + p)     (c*1 is exact)
// i.e. 2 packed instructions per 2 MACs instead of 4 scalar FMUL/FADD.
// The constants come in as kernel arguments so ptxas cannot fold them and
// re-contract the pair into one FFMA2 (it does that with literal constants).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_pipe_probe fp32_pipe_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a);
  unsigned long long rb = *reinterpret_cast<unsigned long long*>(&b);
  unsigned long long rc = *reinterpret_cast<unsigned long long*>(&c);
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(ra), "l"(rb), "l"(rc));
  return *reinterpret_cast<float2*>(&d);
}

template <int MODE>
__global__ void __launch_bounds__(256) probe(const float* x, float* y, int iters, float2 nz, float2 one) {
  constexpr int C = 16;
  float2 acc[C], b[C];
  for (int i = 0; i < C; ++i) { acc[i] = make_float2(x[i] + threadIdx.x, x[i + 1]); b[i] = make_float2(x[i + 20], x[i + 21]); }
  float2 a = make_float2(x[40], x[41]);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i) {
      if constexpr (MODE == 0) {  // scalar FFMA
        acc[i].x = __fmaf_rn(a.x, acc[i].x, b[i].x);
        acc[i].y = __fmaf_rn(a.y, acc[i].y, b[i].y);
      } else if constexpr (MODE == 1) {  // scalar FMUL + FADD
        acc[i].x = __fadd_rn(__fmul_rn(a.x, acc[i].x), b[i].x);
        acc[i].y = __fadd_rn(__fmul_rn(a.y, acc[i].y), b[i].y);
      } else if constexpr (MODE == 2) {  // packed FFMA2
        acc[i] = ffma2(a, acc[i], b[i]);
      } else {  // exact via two FFMA2
        float2 p = ffma2(a, acc[i], nz);
        acc[i] = ffma2(p, one, b[i]);
      }
    }
  }
  float s = 0.f;
  for (int i = 0; i < C; ++i) s += acc[i].x + acc[i].y;
  if (s == 1234.5f) y[threadIdx.x] = s;
}

template <int MODE>
double run(const float* x, float* y, int iters, int blocks) {
  float2 nz = make_float2(-0.0f, -0.0f), one = make_float2(1.f, 1.f);
  probe<MODE><<<blocks, 256>>>(x, y, 64, nz, one);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<MODE><<<blocks, 256>>>(x, y, iters, nz, one);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double macs = 32.0 * iters * 256.0 * blocks;  // 16 float2 chains = 32 MACs per iter per thread
  return 2 * macs / (ms * 1e-3) / 1e12;
}

int main() {
  float *x, *y;
  cudaMalloc(&x, 4096); cudaMalloc(&y, 4096);
  cudaMemset(x, 0, 4096);
  const int iters = 1 << 15, blocks = 148 * 8;
  printf("ffma_scalar %.1f\n", run<0>(x, y, iters, blocks));
  printf("fmul_fadd_scalar %.1f\n", run<1>(x, y, iters, blocks));
  printf("ffma2 %.1f\n", run<2>(x, y, iters, blocks));
  printf("exact_2xffma2 %.1f\n", run<3>(x, y, iters, blocks));
  printf("ffma_scalar %.1f\n", run<0>(x, y, iters, blocks));
  printf("exact_2xffma2 %.1f\n", run<3>(x, y, iters, blocks));
  return 0;
}
