// tcgen05 / TMEM tensor-core im2win convolution (TF32 or BF16 operands, FP32 accumulate).
//
// Same GEMM as the FP32 kernel (winconv kernels/optimized.py:66-214,
// reference.py:30-46) re-mapped onto the 5th-generation tensor cores:
//   D[pixel n][co m] = sum_k' A[n][k'] * B[m][k']
//   * UMMA M = 128 pixels (one TMEM lane per pixel), UMMA N = a Co tile
//     (64/96/128/256), accumulators in TMEM, double buffered so the epilogue
//     of tile i overlaps the MMAs of tile i+1;
//   * the K axis is re-ordered per channel to the im2win window order,
//     k' = c*Hf*Wf + fw*Hf + fh, so A[n][c-run] is the *contiguous* window
//     Ĩ[src_off(n) + c*Ho*RL + 0 .. Hf*Wf-1] (layouts.py:187-199 shows the
//     window slice is contiguous); the filter is packed in the same order;
//   * the filter tile (B, K-major) arrives by TMA with 128-byte swizzle;
//   * the window tile (A, K-major, 128-byte swizzle) is gathered by 8
//     producer warps straight from Ĩ (LDG -> round to tf32 / convert to bf16
//     -> STS in the UMMA canonical layout -> fence.proxy.async -> mbarrier);
//   * one elected thread issues tcgen05.mma; tcgen05.commit releases smem
//     stages and signals the epilogue;
//   * 4 epilogue warps: tcgen05.ld (32 lanes x 16 columns) -> coalesced NCHW
//     stores (consecutive lanes = consecutive output pixels).
// Persistent: one CTA per SM walks a static tile schedule.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "tc_common.cuh"

namespace im2win {
namespace tc {

constexpr int kProducerWarps = 8;
constexpr int kEpilogueWarp0 = 4;  // warps 4..7 (warp % 4 == TMEM lane quarter)
constexpr int kProducerWarp0 = 8;  // warps 8..15
constexpr int kThreads = (kProducerWarp0 + kProducerWarps) * 32;

struct TcArgs {
  const float* __restrict__ win;   // Ĩ, fp32
  const int* __restrict__ delta;   // [Kp] window offset of k' within an image's Ĩ, -1 = padding
  float* __restrict__ out;         // (N, Co, Ho, Wo)
  uint32_t n_gemm;                 // N*Ho*Wo
  uint32_t c_in, h_out, w_out, row_len, s_hf, hw;
  uint32_t co;                     // real Co
  uint32_t k_slabs;                // Kp / BK
  uint32_t pix_tiles, co_tiles;
  FastDiv fd_hw, fd_wo;
};

// ---------------------------------------------------------------- the kernel
template <bool BF16, int N, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    conv_tc_kernel(const TcArgs a, const __grid_constant__ CUtensorMap tmap_b) {
  constexpr uint32_t kABytes = kTileM * kRowBytes;  // 16 KB
  constexpr uint32_t kBBytes = N * kRowBytes;
  constexpr uint32_t kStageBytes = kABytes + kBBytes;
  constexpr int kBK = BF16 ? 64 : 32;             // K elements per stage (one 128 B row)
  constexpr int kUK = BF16 ? 16 : 8;              // K per tcgen05.mma
  constexpr uint32_t kTmemCols = (2 * N <= 128) ? 128 : (2 * N <= 256 ? 256 : 512);
  constexpr uint32_t kIdesc = instr_desc<BF16, N>();

  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2];
  __shared__ __align__(8) uint64_t tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], kProducerWarps + 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4);
    }
    fence_barrier_init();
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmap_b) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  const uint32_t total_tiles = a.pix_tiles * a.co_tiles;

  if (warp == 0) {
    // ---------------- TMA producer for the filter tile (B) ----------------
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (uint32_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const int co_blk = t % a.co_tiles;
        for (uint32_t ks = 0; ks < a.k_slabs; ++ks) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* bdst = smem + stage * kStageBytes + kABytes;
          mbar_arrive_expect_tx(&full_bar[stage], kBBytes);
          tma_load_2d(bdst, &tmap_b, &full_bar[stage], ks * kBK, co_blk * N);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (single thread) ----------------
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      uint32_t acc = 0, acc_phase = 0;
      for (uint32_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * N;
        for (uint32_t ks = 0; ks < a.k_slabs; ++ks) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t abase = smem_u32(smem + stage * kStageBytes);
          const uint32_t bbase = abase + kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / kUK; ++kk) {
            // advancing K inside the 128 B swizzle row = +32 B on the start address
            const uint64_t ad = smem_desc_sw128(abase + kk * 32);
            const uint64_t bd = smem_desc_sw128(bbase + kk * 32);
            mma<BF16>(tmem_d, ad, bd, kIdesc, (ks | kk) != 0);
          }
          mma_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull_bar[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= kEpilogueWarp0 && warp < kEpilogueWarp0 + 4) {
    // ---------------- epilogue: TMEM -> registers -> NCHW ----------------
    const int quarter = warp % 4;  // TMEM lanes [32*quarter, +32)
    uint32_t acc = 0, acc_phase = 0;
    for (uint32_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      const uint32_t co_blk = t % a.co_tiles;
      const uint32_t pix_blk = t / a.co_tiles;
      const uint32_t n = pix_blk * kTileM + quarter * 32 + lane;
      const bool valid = n < a.n_gemm;
      int64_t obase = 0;
      if (valid) {
        uint32_t img, rem;
        a.fd_hw.divmod(n, img, rem);
        obase = static_cast<int64_t>(img) * a.co * a.hw + rem;
      }
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * N;
#pragma unroll
      for (int j0 = 0; j0 < N; j0 += 16) {
        uint32_t r[16];
        tmem_ld16(taddr + j0, r);
        const uint32_t m0 = co_blk * N + j0;
        if (valid) {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (m0 + q < a.co) a.out[obase + static_cast<int64_t>(m0 + q) * a.hw] = __uint_as_float(r[q]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= kProducerWarp0) {
    // ---------------- window-tile producers: Ĩ -> swizzled A stage ----------------
    // Warp pw owns A rows [16*pw, 16*pw+16) of every tile; lane = position in the
    // 128-byte K row.  Row r, K-byte b lives at (r/8)*1024 + (r%8)*128 + ((b/16)^(r%8))*16 + b%16
    // (UMMA K-major SWIZZLE_128B canonical layout).
    const int pw = warp - kProducerWarp0;
    constexpr int kRows = kTileM / kProducerWarps;
    auto row_offset = [&](uint32_t t) -> int64_t {
      int64_t off = -1;
      if (lane < kRows) {
        const uint32_t n = (t / a.co_tiles) * kTileM + pw * kRows + lane;
        if (n < a.n_gemm) {
          uint32_t img, rem, oh, ow;
          a.fd_hw.divmod(n, img, rem);
          a.fd_wo.divmod(rem, oh, ow);
          off = (static_cast<int64_t>(img) * a.c_in * a.h_out + oh) * a.row_len + static_cast<int64_t>(ow) * a.s_hf;
        }
      }
      return off;
    };
    auto a_slot = [&](uint32_t stage_idx, int i) -> uint8_t* {
      const int r = pw * kRows + i;
      const uint32_t chunk = (static_cast<uint32_t>(lane) >> 2) ^ (r & 7);
      return smem + stage_idx * kStageBytes + (r >> 3) * 1024 + (r & 7) * 128 + chunk * 16 + (lane & 3) * 4;
    };
    if constexpr (!BF16) {
      // TF32: 4-byte cp.async straight into the swizzled slot (tf32 = fp32 bits, the
      // tensor core ignores the low mantissa: round-toward-zero); D slabs in flight per warp.
      constexpr int D = STAGES >= 5 ? 4 : STAGES - 1;
      uint32_t stage = 0, phase = 0, rstage = 0, unretired = 0;
      for (uint32_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const int64_t my_off = row_offset(t);
        for (uint32_t ks = 0; ks < a.k_slabs; ++ks) {
          const int d = __ldg(a.delta + ks * kBK + lane);
          mbar_wait(&empty_bar[stage], phase ^ 1);
#pragma unroll
          for (int i = 0; i < kRows; ++i) {
            const int64_t off = __shfl_sync(0xffffffffu, my_off, i);
            const bool zero = off < 0 || d < 0;
            cp_async_4_zfill(smem_u32(a_slot(stage, i)), zero ? a.win : a.win + off + d, zero);
          }
          cp_async_commit();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          if (++unretired == D + 1) {
            cp_async_wait<D>();
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&full_bar[rstage]);
            if (++rstage == STAGES) rstage = 0;
            --unretired;
          }
        }
      }
      cp_async_wait<0>();
      fence_proxy_async_smem();
      __syncwarp();
      for (; unretired > 0; --unretired) {
        if (lane == 0) mbar_arrive(&full_bar[rstage]);
        if (++rstage == STAGES) rstage = 0;
      }
    } else {
      // BF16: registers (fp32 -> bf16x2), software pipelined one slab ahead.
      uint32_t stage = 0, phase = 0;
      uint32_t t = blockIdx.x, ks = 0;
      int64_t my_off = t < total_tiles ? row_offset(t) : -1;
      float c0[kRows], c1[kRows];
      auto load = [&](uint32_t kslab, int64_t off_reg, float (&v0)[kRows], float (&v1)[kRows]) {
        const int2 dd = __ldg(reinterpret_cast<const int2*>(a.delta + kslab * kBK) + lane);
#pragma unroll
        for (int i = 0; i < kRows; ++i) {
          const int64_t off = __shfl_sync(0xffffffffu, off_reg, i);
          v0[i] = (off >= 0 && dd.x >= 0) ? __ldg(a.win + off + dd.x) : 0.0f;
          v1[i] = (off >= 0 && dd.y >= 0) ? __ldg(a.win + off + dd.y) : 0.0f;
        }
      };
      if (t < total_tiles) load(0, my_off, c0, c1);
      while (t < total_tiles) {
        uint32_t nt = t, nks = ks + 1;
        if (nks == a.k_slabs) { nks = 0; nt += gridDim.x; }
        float n0[kRows], n1[kRows];
        if (nt < total_tiles) {
          if (nt != t) my_off = row_offset(nt);
          load(nks, my_off, n0, n1);
        }
        mbar_wait(&empty_bar[stage], phase ^ 1);
#pragma unroll
        for (int i = 0; i < kRows; ++i) *reinterpret_cast<uint32_t*>(a_slot(stage, i)) = pack_bf16x2(c0[i], c1[i]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_bar[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
#pragma unroll
        for (int i = 0; i < kRows; ++i) { c0[i] = n0[i]; c1[i] = n1[i]; }
        t = nt;
        ks = nks;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

// ---------------------------------------------------------------- packing
// B[m][k'] = F[m][c][fh][fw] with k' = c*Hf*Wf + fw*Hf + fh (zero padded to Mp x Kp);
// delta[k'] = c*chan_stride + (k' mod Hf*Wf), -1 for k' >= K.
template <bool BF16>
__global__ void pack_filter_tc_kernel(const float* __restrict__ flt, void* __restrict__ packed, int* __restrict__ delta,
                                      int M, int K, int Mp, int Kp, int h_f, int w_f, int chan_stride) {
  const int fhw = h_f * w_f;
  const int64_t total = static_cast<int64_t>(Mp) * Kp;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i / Kp);
    const int kp = static_cast<int>(i % Kp);
    float v = 0.0f;
    if (m < M && kp < K) {
      const int c = kp / fhw, j = kp % fhw;
      const int fw = j / h_f, fh = j % h_f;
      v = flt[(static_cast<int64_t>(m) * K) + (c * h_f + fh) * w_f + fw];
    }
    if constexpr (BF16) {
      reinterpret_cast<__nv_bfloat16*>(packed)[i] = __float2bfloat16_rn(v);
    } else {
      uint32_t r;
      asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(v));
      reinterpret_cast<uint32_t*>(packed)[i] = r;
    }
    if (m == 0) delta[kp] = kp < K ? (kp / fhw) * chan_stride + (kp % fhw) : -1;
  }
}

// ---------------------------------------------------------------- host side
template <bool BF16, int N, int STAGES>
static int launch(const TcArgs& a0, void* packed, int Kp, int Mp, cudaStream_t stream, const char** err) {
  TcArgs a = a0;
  constexpr int kBK = BF16 ? 64 : 32;
  a.k_slabs = Kp / kBK;
  a.co_tiles = Mp / N;
  CUtensorMap map;
  auto enc = get_encode_fn();
  if (!enc) {
    *err = "conv_tc: cuTensorMapEncodeTiled unavailable";
    return 2;
  }
  const cuuint64_t esz = BF16 ? 2 : 4;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(Mp)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(Kp) * esz};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(N)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&map, BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, packed, dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "conv_tc: cuTensorMapEncodeTiled failed";
    return 2;
  }
  const size_t smem = static_cast<size_t>(STAGES) * (kTileM + N) * kRowBytes + 1024;
  auto kern = conv_tc_kernel<BF16, N, STAGES>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 2;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t tiles = a.pix_tiles * a.co_tiles;
  const uint32_t grid = tiles < static_cast<uint32_t>(sms) ? tiles : static_cast<uint32_t>(sms);
  im2win_note_kernel("conv_tc_kernel (gathered reference window tiles)");
  kern<<<grid, kThreads, smem, stream>>>(a, map);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 2;
  }
  return 0;
}

static int pick_n(int64_t co) {
  if (co <= 64) return 64;
  if (co <= 96) return 96;
  if (co <= 128) return 128;
  return 256;
}

}  // namespace tc
}  // namespace im2win

size_t im2win_tc_workspace_bytes(int64_t c_out, int64_t K, int variant) {
  (void)variant;
  const int64_t Mp = (c_out + 255) / 256 * 256 + 256;
  const int64_t Kp = (K + 63) / 64 * 64;
  return static_cast<size_t>(Mp * Kp) * 4 + static_cast<size_t>(Kp) * 4 + 1024;
}

int im2win_launch_conv_tc(const float* win, const float* flt, float* out, void* workspace, int64_t n, int64_t c_in,
                          int64_t c_out, int64_t h_out, int64_t w_out, int64_t row_len, int h_f, int w_f, int stride,
                          int variant, int cfg, cudaStream_t stream, const char** err) {
  using namespace im2win;
  using namespace im2win::tc;
  (void)cfg;
  const bool bf16 = variant == 3;
  const int64_t K = c_in * h_f * w_f;
  const int64_t hw = h_out * w_out;
  const int64_t n_gemm = n * hw;
  if (n_gemm >= (1ll << 31) || K >= (1ll << 24) || c_in * h_out * row_len >= (1ll << 31)) {
    *err = "im2win_conv_f32: extents exceed the kernel's index range";
    return 1;
  }
  const int N = pick_n(c_out);
  const int bk = bf16 ? 64 : 32;
  const int Kp = static_cast<int>((K + bk - 1) / bk * bk);
  const int Mp = static_cast<int>((c_out + N - 1) / N * N);
  const size_t esz = bf16 ? 2 : 4;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  void* packed = ws;
  int* delta = reinterpret_cast<int*>(ws + ((static_cast<size_t>(Mp) * Kp * esz + 255) & ~size_t(255)));
  if (bf16)
    pack_filter_tc_kernel<true><<<256, 256, 0, stream>>>(flt, packed, delta, static_cast<int>(c_out), static_cast<int>(K),
                                                         Mp, Kp, h_f, w_f, static_cast<int>(h_out * row_len));
  else
    pack_filter_tc_kernel<false><<<256, 256, 0, stream>>>(flt, packed, delta, static_cast<int>(c_out), static_cast<int>(K),
                                                          Mp, Kp, h_f, w_f, static_cast<int>(h_out * row_len));
  TcArgs a{};
  a.win = win;
  a.delta = delta;
  a.out = out;
  a.n_gemm = static_cast<uint32_t>(n_gemm);
  a.c_in = static_cast<uint32_t>(c_in);
  a.h_out = static_cast<uint32_t>(h_out);
  a.w_out = static_cast<uint32_t>(w_out);
  a.row_len = static_cast<uint32_t>(row_len);
  a.s_hf = static_cast<uint32_t>(stride * h_f);
  a.hw = static_cast<uint32_t>(hw);
  a.co = static_cast<uint32_t>(c_out);
  a.pix_tiles = static_cast<uint32_t>((n_gemm + kTileM - 1) / kTileM);
  a.fd_hw = FastDiv(static_cast<uint32_t>(hw));
  a.fd_wo = FastDiv(static_cast<uint32_t>(w_out));
#define IM2WIN_TC(BF, NN, ST) return launch<BF, NN, ST>(a, packed, Kp, Mp, stream, err)
  if (bf16) {
    switch (N) {
      case 64: IM2WIN_TC(true, 64, 8);
      case 96: IM2WIN_TC(true, 96, 6);
      case 128: IM2WIN_TC(true, 128, 6);
      default: IM2WIN_TC(true, 256, 4);
    }
  } else {
    switch (N) {
      case 64: IM2WIN_TC(false, 64, 8);
      case 96: IM2WIN_TC(false, 96, 6);
      case 128: IM2WIN_TC(false, 128, 6);
      default: IM2WIN_TC(false, 256, 4);
    }
  }
#undef IM2WIN_TC
}
