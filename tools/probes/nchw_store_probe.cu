// Does the TC epilogue's NCHW store pattern (lane = pixel, one 4-byte store per channel,
// tiles of box_w pixels x 64 channels) limit conv7-shaped outputs?  Writes N x 64 x 222 x 222
// fp32 with that pattern from 148 persistent CTAs (warps = lane quarters x column halves,
// as in the kernels), and with a plain grid-stride float4 fill, and reports TB/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nchw_store_probe nchw_store_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) pattern(float* out, int n, int co, int ho, int wo, int box_w, int warps_per_tile) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int quarter = warp % 4, half = warp / 4;  // 8 warps: 4 lane quarters x 2 column halves
  const int ow_tiles = (wo + box_w - 1) / box_w;
  const long long tiles = (long long)n * ho * ow_tiles;
  const int r = quarter * 32 + lane;
  const long long hw = (long long)ho * wo;
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int owt = t % ow_tiles;
    const long long rest = t / ow_tiles;
    const int oh = rest % ho;
    const long long img = rest / ho;
    const int ow = owt * box_w + r;
    if (r < box_w && ow < wo) {
      float* base = out + img * co * hw + (long long)oh * wo + ow;
      const int c0 = half * (co / 2);
#pragma unroll 8
      for (int c = 0; c < co / 2; ++c) base[(long long)(c0 + c) * hw] = (float)c;
    }
  }
}

// Variant: plane stride padded by `pad_elems` floats (is it L2/DRAM address aliasing of the 64 planes?)
__global__ void __launch_bounds__(256) pattern_pad(float* out, int n, int co, int ho, int wo, int box_w, long long plane) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int quarter = warp % 4, half = warp / 4;
  const int ow_tiles = (wo + box_w - 1) / box_w;
  const long long tiles = (long long)n * ho * ow_tiles;
  const int r = quarter * 32 + lane;
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int owt = t % ow_tiles;
    const long long rest = t / ow_tiles;
    const int oh = rest % ho;
    const long long img = rest / ho;
    const int ow = owt * box_w + r;
    if (r < box_w && ow < wo) {
      float* base = out + img * co * plane + (long long)oh * wo + ow;
      const int c0 = half * (co / 2);
#pragma unroll 8
      for (int c = 0; c < co / 2; ++c) base[(long long)(c0 + c) * plane] = (float)c;
    }
  }
}

// Variant: each warp writes one plane's 128-pixel run per step with 4 consecutive pixels per lane
__global__ void __launch_bounds__(256) pattern_runs(float* out, int n, int co, int ho, int wo, int box_w) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int ow_tiles = (wo + box_w - 1) / box_w;
  const long long tiles = (long long)n * ho * ow_tiles;
  const long long hw = (long long)ho * wo;
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int owt = t % ow_tiles;
    const long long rest = t / ow_tiles;
    const int oh = rest % ho;
    const long long img = rest / ho;
    for (int c = warp; c < co; c += 8) {
      float* base = out + (img * co + c) * hw + (long long)oh * wo + owt * box_w;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int px = q * 32 + lane;
        if (px < box_w && owt * box_w + px < wo) base[px] = (float)c;
      }
    }
  }
}

// Variant: a "tile" is `rows_per` full output rows; each warp writes one plane's contiguous run
// of rows_per * wo pixels (NCHW rows are contiguous within a plane).
__global__ void __launch_bounds__(256) pattern_rowruns(float* out, int n, int co, int ho, int wo, int rows_per) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int oh_tiles = (ho + rows_per - 1) / rows_per;
  const long long tiles = (long long)n * oh_tiles;
  const long long hw = (long long)ho * wo;
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int oh0 = (t % oh_tiles) * rows_per;
    const long long img = t / oh_tiles;
    const int run = min(rows_per, ho - oh0) * wo;
    for (int c = warp; c < co; c += 8) {
      float* base = out + (img * co + c) * hw + (long long)oh0 * wo;
      for (int px = lane; px < run; px += 32) base[px] = (float)c;
    }
  }
}

// Variant: the kernels' pattern with a store cache hint (0: default, 1: .cs streaming, 2: L2 evict_last)
template <int HINT>
__global__ void __launch_bounds__(256) pattern_hint(float* out, int n, int co, int ho, int wo, int box_w) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int quarter = warp % 4, half = warp / 4;
  const int ow_tiles = (wo + box_w - 1) / box_w;
  const long long tiles = (long long)n * ho * ow_tiles;
  const int r = quarter * 32 + lane;
  const long long hw = (long long)ho * wo;
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int owt = t % ow_tiles;
    const long long rest = t / ow_tiles;
    const int oh = rest % ho;
    const long long img = rest / ho;
    const int ow = owt * box_w + r;
    if (r < box_w && ow < wo) {
      float* base = out + img * co * hw + (long long)oh * wo + ow;
      const int c0 = half * (co / 2);
#pragma unroll 8
      for (int c = 0; c < co / 2; ++c) {
        float* d = base + (long long)(c0 + c) * hw;
        if (HINT == 1) __stcs(d, (float)c);
        else if (HINT == 2) asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(d), "f"((float)c), "l"(pol) : "memory");
        else *d = (float)c;
      }
    }
  }
}

// Variant: the tile (box_w pixels x co planes) staged in smem, then each plane's run leaves by
// one TMA bulk store (16-byte aligned middle) + plain stores for the unaligned ends.
__global__ void __launch_bounds__(256) pattern_bulk(float* out, int n, int co, int ho, int wo, int box_w) {
  extern __shared__ __align__(128) float stg[];  // [2][co][box_w + 4]
  const int pitch = (box_w + 4 + 3) / 4 * 4;
  const int ow_tiles = (wo + box_w - 1) / box_w;
  const long long tiles = (long long)n * ho * ow_tiles;
  const long long hw = (long long)ho * wo;
  int it = 0;
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
    const int owt = t % ow_tiles;
    const long long rest = t / ow_tiles;
    const int oh = rest % ho;
    const long long img = rest / ho;
    const int ow0 = owt * box_w;
    const int run = min(box_w, wo - ow0);
    float* sb = stg + (it & 1) * co * pitch;
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    const long long base0 = img * co * hw + (long long)oh * wo + ow0;
    const int head = (4 - (int)(base0 & 3)) & 3;  // same for every plane when hw % 4 == 0
    for (int i = threadIdx.x; i < co * run; i += blockDim.x) {
      const int c = i / run, px = i % run;
      sb[c * pitch + ((head == 0 ? 0 : 4 - head) + px)] = (float)c;  // shift so aligned globals land on aligned smem
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const int sh = head == 0 ? 0 : 4 - head;
    const int mid = ((run - head) / 4) * 4;
    for (int c = threadIdx.x / 32; c < co; c += blockDim.x / 32) {
      float* dst = out + base0 + (long long)c * hw;
      const float* src = sb + c * pitch + sh;
      const int lane = threadIdx.x % 32;
      if (lane < head) dst[lane] = src[lane];
      if (lane < run - head - mid) dst[head + mid + lane] = src[head + mid + lane];
      if (lane == 0 && mid > 0)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + head),
                     "r"((unsigned)__cvta_generic_to_shared(src + head)), "r"(mid * 4) : "memory");
    }
    if (threadIdx.x % 32 == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Variant: the kernels' lane-per-pixel pattern, but each CTA takes `group` consecutive tiles
// (e.g. both halves of an output row) back to back instead of striding by gridDim.x
__global__ void __launch_bounds__(256) pattern_grouped(float* out, int n, int co, int ho, int wo, int box_w, int group) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int quarter = warp % 4, half = warp / 4;
  const int ow_tiles = (wo + box_w - 1) / box_w;
  const long long tiles = (long long)n * ho * ow_tiles;
  const int r = quarter * 32 + lane;
  const long long hw = (long long)ho * wo;
  for (long long t0 = (long long)blockIdx.x * group; t0 < tiles; t0 += (long long)gridDim.x * group) {
    for (long long t = t0; t < t0 + group && t < tiles; ++t) {
      const int owt = t % ow_tiles;
      const long long rest = t / ow_tiles;
      const int oh = rest % ho;
      const long long img = rest / ho;
      const int ow = owt * box_w + r;
      if (r < box_w && ow < wo) {
        float* base = out + img * co * hw + (long long)oh * wo + ow;
        const int c0 = half * (co / 2);
#pragma unroll 8
        for (int c = 0; c < co / 2; ++c) base[(long long)(c0 + c) * hw] = (float)c;
      }
    }
  }
}

// Variant: the TC epilogue staged through shared memory -- 8 warps, warp w owning lane quarter
// w % 4 (32 pixels) and channel half w / 4 of a `group`-tile run (both halves of an output row
// for group 2); each warp writes its values into smem [co][group*box_w] (lane = pixel), one
// barrier, then warp w writes channel rows c = w, w+8, ... as whole runs (lane = pixel,
// consecutive 128-byte pieces of the same plane row back to back).
__global__ void __launch_bounds__(256) pattern_staged(float* out, int n, int co, int ho, int wo, int box_w, int group) {
  extern __shared__ float stg[];  // [co][group * box_w]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int quarter = warp % 4, half = warp / 4;
  const int ow_tiles = (wo + box_w - 1) / box_w;
  const long long tiles = (long long)n * ho * ow_tiles;
  const int r = quarter * 32 + lane;
  const int pitch = group * box_w;
  const long long hw = (long long)ho * wo;
  for (long long t0 = (long long)blockIdx.x * group; t0 < tiles; t0 += (long long)gridDim.x * group) {
    // stage: like tcgen05.ld -> st.shared, per tile of the run
    for (int g = 0; g < group && t0 + g < tiles; ++g) {
      if (r < box_w) {
        const int c0 = half * (co / 2);
#pragma unroll 8
        for (int c = 0; c < co / 2; ++c) stg[(c0 + c) * pitch + g * box_w + r] = (float)(c0 + c);
      }
    }
    __syncthreads();
    // write: the run's pixels are consecutive in each plane (group tiles = whole rows)
    const int owt = t0 % ow_tiles;
    const long long rest = t0 / ow_tiles;
    const int oh = rest % ho;
    const long long img = rest / ho;
    const int run = min(pitch, wo - owt * box_w);
    for (int c = warp; c < co; c += 8) {
      float* base = out + (img * co + c) * hw + (long long)oh * wo + owt * box_w;
      for (int px = lane; px < run; px += 32) base[px] = stg[c * pitch + px];
    }
    __syncthreads();
  }
}

// Variant: 8 stager warps (the TC epilogue: lane = pixel values into smem [co][2*box_w], both
// halves of an output row) and 8 writer warps that only copy staged rows out (channel rows as
// whole runs, lane = pixel), double-buffered with mbarriers so the writers never wait on a
// barrier the stagers hold.
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(unsigned long long* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* b, unsigned ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(
                   su32(b)), "r"(ph) : "memory");
}
__global__ void __launch_bounds__(512) pattern_writers(float* out, int n, int co, int ho, int wo, int box_w) {
  extern __shared__ float stg[];  // [2][co][2 * box_w]
  __shared__ unsigned long long full[2], empty[2];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int pitch = 2 * box_w;
  const long long rows = (long long)n * ho;
  const long long hw = (long long)ho * wo;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) { bar_init(&full[b], 8); bar_init(&empty[b], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int it = 0;
  if (warp < 8) {  // stagers
    const int quarter = warp % 4, half = warp / 4;
    for (long long row = blockIdx.x; row < rows; row += gridDim.x, ++it) {
      const int b = it & 1;
      if (it >= 2) bar_wait(&empty[b], ((it >> 1) - 1) & 1);
      float* sb = stg + b * co * pitch;
      for (int g = 0; g < 2; ++g) {
        const int r = quarter * 32 + lane;
        if (r < box_w) {
          const int c0 = half * (co / 2);
#pragma unroll 8
          for (int c = 0; c < co / 2; ++c) sb[(c0 + c) * pitch + g * box_w + r] = (float)(c0 + c);
        }
      }
      __syncwarp();
      if (lane == 0) bar_arrive(&full[b]);
    }
  } else {  // writers
    const int ww = warp - 8;
    for (long long row = blockIdx.x; row < rows; row += gridDim.x, ++it) {
      const int b = it & 1;
      bar_wait(&full[b], (it >> 1) & 1);
      const float* sb = stg + b * co * pitch;
      const int oh = row % ho;
      const long long img = row / ho;
      for (int c = ww; c < co; c += 8) {
        float* base = out + (img * co + c) * hw + (long long)oh * wo;
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = (q * 32 + lane < wo) ? sb[c * pitch + q * 32 + lane] : 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q * 32 + lane < wo) base[q * 32 + lane] = v[q];
      }
      __syncwarp();
      if (lane == 0) bar_arrive(&empty[b]);
    }
  }
}

__global__ void fill(float4* out, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
    out[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}

int main() {
  const int n = 128, co = 64, ho = 222, wo = 222;
  const size_t elems = (size_t)n * co * ho * wo;
  float* out;
  cudaMalloc(&out, elems * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int box_w : {111, 128, 74}) {
    pattern<<<148, 256>>>(out, n, co, ho, wo, box_w, 8);
    cudaEventRecord(e0);
    pattern<<<148, 256>>>(out, n, co, ho, wo, box_w, 8);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("pattern box_w=%d: %.3f ms  %.2f TB/s\n", box_w, ms, elems * 4 / (ms * 1e-3) / 1e12);
  }
  for (int ctas : {148, 148 * 2, 148 * 8}) {
    pattern<<<ctas, 256>>>(out, n, co, ho, wo, 111, 8);
    cudaEventRecord(e0);
    pattern<<<ctas, 256>>>(out, n, co, ho, wo, 111, 8);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("pattern ctas=%d: %.3f ms  %.2f TB/s\n", ctas, ms, elems * 4 / (ms * 1e-3) / 1e12);
  }
  {
    const long long plane = (long long)ho * wo;
    float* out2;
    cudaMalloc(&out2, ((size_t)n * co * (plane + 64)) * 4);
    for (long long pad : {0LL, 32LL, 64LL}) {
      pattern_pad<<<148, 256>>>(out2, n, co, ho, wo, 111, plane + pad);
      cudaEventRecord(e0);
      pattern_pad<<<148, 256>>>(out2, n, co, ho, wo, 111, plane + pad);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("pattern plane+%lld: %.3f ms  %.2f TB/s\n", pad, ms, elems * 4 / (ms * 1e-3) / 1e12);
    }
    cudaFree(out2);
  }
  for (int box_w : {111, 128}) {
    pattern_runs<<<148, 256>>>(out, n, co, ho, wo, box_w);
    cudaEventRecord(e0);
    pattern_runs<<<148, 256>>>(out, n, co, ho, wo, box_w);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("runs box_w=%d: %.3f ms  %.2f TB/s\n", box_w, ms, elems * 4 / (ms * 1e-3) / 1e12);
  }
  for (int rp : {1, 2, 4, 8}) {
    pattern_rowruns<<<148, 256>>>(out, n, co, ho, wo, rp);
    cudaEventRecord(e0);
    pattern_rowruns<<<148, 256>>>(out, n, co, ho, wo, rp);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("rowruns rows=%d: %.3f ms  %.2f TB/s\n", rp, ms, elems * 4 / (ms * 1e-3) / 1e12);
  }
  {
    float ms;
    pattern_hint<1><<<148, 256>>>(out, n, co, ho, wo, 111);
    cudaEventRecord(e0); pattern_hint<1><<<148, 256>>>(out, n, co, ho, wo, 111); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("pattern .cs: %.3f ms  %.2f TB/s\n", ms, elems * 4 / (ms * 1e-3) / 1e12);
    pattern_hint<2><<<148, 256>>>(out, n, co, ho, wo, 111);
    cudaEventRecord(e0); pattern_hint<2><<<148, 256>>>(out, n, co, ho, wo, 111); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("pattern evict_last: %.3f ms  %.2f TB/s\n", ms, elems * 4 / (ms * 1e-3) / 1e12);
  }
  {
    float ms;
    for (int bw : {111, 222}) {
      const size_t sm = 2ull * co * ((bw + 7) / 4 * 4) * 4;
      cudaFuncSetAttribute(pattern_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      pattern_bulk<<<148, 256, sm>>>(out, n, co, ho, wo, bw);
      cudaEventRecord(e0); pattern_bulk<<<148, 256, sm>>>(out, n, co, ho, wo, bw); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      printf("bulk box_w=%d: %.3f ms  %.2f TB/s  (%s)\n", bw, ms, elems * 4 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int g : {1, 2, 4, 8}) {
    float ms;
    pattern_grouped<<<148, 256>>>(out, n, co, ho, wo, 111, g);
    cudaEventRecord(e0); pattern_grouped<<<148, 256>>>(out, n, co, ho, wo, 111, g); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("grouped box_w=111 group=%d: %.3f ms  %.2f TB/s\n", g, ms, elems * 4 / (ms * 1e-3) / 1e12);
  }
  for (int g : {1, 2}) {
    float ms;
    const size_t sm = (size_t)co * g * 111 * 4;
    cudaFuncSetAttribute(pattern_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    pattern_staged<<<148, 256, sm>>>(out, n, co, ho, wo, 111, g);
    cudaEventRecord(e0); pattern_staged<<<148, 256, sm>>>(out, n, co, ho, wo, 111, g); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("staged box_w=111 group=%d: %.3f ms  %.2f TB/s (%s)\n", g, ms, elems * 4 / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  }
  {
    float ms;
    const size_t sm = 2ull * co * 2 * 111 * 4;
    cudaFuncSetAttribute(pattern_writers, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    pattern_writers<<<148, 512, sm>>>(out, n, co, ho, wo, 111);
    cudaEventRecord(e0); pattern_writers<<<148, 512, sm>>>(out, n, co, ho, wo, 111); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("writers (8 stagers + 8 row writers, double buffer): %.3f ms  %.2f TB/s (%s)\n", ms,
           elems * 4 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  fill<<<148 * 8, 256>>>((float4*)out, elems / 4);
  cudaEventRecord(e0);
  fill<<<148 * 8, 256>>>((float4*)out, elems / 4);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("float4 fill: %.3f ms  %.2f TB/s\n", ms, elems * 4 / (ms * 1e-3) / 1e12);
  return 0;
}
