// UMMA issue-rate probe (B200): back-to-back tcgen05.mma from fixed shared-memory tiles,
// one CTA per SM, for M = 128 with N = 64/128/256 (cta_group::1) and M = 256 (cta_group::2),
// BF16 and TF32; also "A reuse" (the same A with MT accumulators, as the phase kernel) and the
// A tile advanced by one 128-byte row (the phase/shift kernels' shifted descriptors).
// Prints achieved TFLOP/s per configuration (whole chip).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2306_14316_b200/csrc -o umma_rate umma_rate.cu -lcuda
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_common.cuh"

using namespace im2win;
using namespace im2win::tc;

template <bool BF16, int N, bool PAIR, int SHIFT>
__global__ void __launch_bounds__(128, 1) umma_probe(int iters, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t tmem_sh;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kUK = BF16 ? 16 : 8;
  constexpr int kBRows = PAIR ? N / 2 : N;
  constexpr uint32_t kA = 136 * 128;
  constexpr uint32_t kIdesc = instr_desc_m<BF16, N, PAIR ? 256 : 128>();
  const int warp = threadIdx.x / 32;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  for (uint32_t i = threadIdx.x; i < (4 * kA + kBRows * 128) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_sh)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_sh)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t abase = smem_u32(smem), bbase = abase + 4 * kA;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t bd = smem_desc_sw128(bbase + kk * 32);
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          const uint64_t ad = smem_desc_sw128(abase + mt * kA + SHIFT * 128 * (kk & 1) + kk * 32);
          if constexpr (PAIR) mma_pair<BF16>(tmem + mt * N % 512, ad, bd, kIdesc, 1);
          else mma<BF16>(tmem + (mt * N) % 512, ad, bd, kIdesc, 1);
        }
      }
    }
    if constexpr (PAIR) mma_commit_pair(&done);
    else mma_commit(&done);
    mbar_wait(&done, 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) cycles[0] = t1 - t0;
  } else if (PAIR && threadIdx.x == 0) {
    mbar_wait(&done, 0);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

template <bool BF16, int N, bool PAIR, int SHIFT>
void run(const char* name) {
  auto kern = umma_probe<BF16, N, PAIR, SHIFT>;
  const size_t smem = 4 * 136 * 128 + 256 * 128 + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  const int iters = 4000;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, iters, cyc);  // warm up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, kern, iters, cyc);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double k = BF16 ? 16 : 8;
  const double flops = 2.0 * (PAIR ? 74 * 256 : 148 * 128) * N * k * 16.0 * iters;
  const double per_mma = static_cast<double>(c) / (16.0 * iters);
  printf("%-34s %s  %7.1f TFLOP/s  %6.1f cycles/MMA\n", name, e == cudaSuccess ? "ok " : cudaGetErrorString(e),
         flops / ms / 1e9, per_mma);
  cudaFree(cyc);
}

int main() {
  run<true, 64, false, 0>("bf16 M128 N64");
  run<true, 64, false, 1>("bf16 M128 N64 A row-shifted");
  run<true, 128, false, 0>("bf16 M128 N128");
  run<true, 256, false, 0>("bf16 M128 N256");
  run<true, 64, true, 0>("bf16 pair M256 N64");
  run<true, 128, true, 0>("bf16 pair M256 N128");
  run<true, 256, true, 0>("bf16 pair M256 N256");
  run<false, 64, false, 0>("tf32 M128 N64");
  run<false, 128, false, 0>("tf32 M128 N128");
  run<false, 256, false, 0>("tf32 M128 N256");
  run<false, 64, true, 0>("tf32 pair M256 N64");
  run<false, 128, true, 0>("tf32 pair M256 N128");
  return 0;
}
