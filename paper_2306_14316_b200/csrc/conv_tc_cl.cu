// Channels-innermost im2win + TMA-fed tcgen05 convolution (the tensor-core fast path).
//
// Layout Ĩcl (internal; the NHWC form of the im2win window layout): for output row
// g = img*Ho + oh, source column col < w_eff, filter row fh < Hf and channel c < C
//     Ĩcl[g][col][fh][c] = X[img][c][oh*s + fh][col]
// It is the reference's window order (layouts.py:73-83: per output row, the Hf input
// rows it touches, column by column, the Hf values of a column contiguous) with the
// channel moved innermost.  A pixel's whole dot-product window is then ONE contiguous
// run of K = Wf*Hf*C elements starting at Ĩcl[g][ow*s][0][0], and consecutive pixels of
// a row are s*Hf*C elements apart, so the GEMM operand
//     A[(g, ow)][k'] = Ĩcl[g*RLc + ow*s*Hf*C + k'],  k' = (fw*Hf + fh)*C + c
// is a strided 3-D view {k', ow, g} that a TMA tensor map walks directly (the windows
// overlap in memory; TMA only reads).  No gather, no repack: TMA delivers 128-byte
// swizzled K-major tiles that tcgen05.mma consumes as-is, K and pixel tails are
// zero-filled by TMA's out-of-bounds handling.
//
// Tile = box_g output rows x box_w output columns (<= 128 pixels = UMMA M rows),
// Co tile = UMMA N.  Warp 0: TMA producer (A + filter B), warp 1: MMA issuer,
// warp 2: TMEM allocator, warps 4-7: epilogue (TMEM -> NCHW, coalesced along ow).
#include <stddef.h>
#include <stdint.h>

#include "tc_common.cuh"

namespace im2win {
namespace tc {

// ---------------------------------------------------------------- transform
// Work unit = (output row g, filter row fh, 32-channel block): the 32 input rows
// X[img][c0..c0+31][oh*s+fh][0..w_eff) are staged in smem (16-byte loads when the
// row pitch allows), then written transposed as Ĩcl[g][col][fh][c0..c0+31] with
// 16-byte (fp32) / 8-byte (bf16) stores.  Smem pitch = 1 mod 32 makes the
// column-wise reads conflict free.  Requires c_in % 4 == 0.
template <bool BF16, bool VEC_IN>
__global__ void __launch_bounds__(256) transform_cl_kernel(const float* __restrict__ src, void* __restrict__ dst,
                                                           uint32_t c_in, uint32_t h_in, uint32_t w_in,
                                                           uint32_t h_out, uint32_t h_f, uint32_t stride,
                                                           uint32_t w_eff, uint32_t c_blocks, uint32_t pitch,
                                                           uint32_t total_units) {
  extern __shared__ float tile[];  // [32][pitch]
  const uint32_t w4 = (w_eff + 3) / 4;
  for (uint32_t u = blockIdx.x; u < total_units; u += gridDim.x) {
    const uint32_t cb = u % c_blocks;
    const uint32_t fh = (u / c_blocks) % h_f;
    const uint32_t g = u / (c_blocks * h_f);
    const uint32_t img = g / h_out, oh = g % h_out;
    const uint32_t c0 = cb * 32;
    const uint32_t nc = min(32u, c_in - c0);
    const float* base = src + ((static_cast<uint64_t>(img) * c_in + c0) * h_in + oh * stride + fh) * w_in;
    const uint64_t chan_stride = static_cast<uint64_t>(h_in) * w_in;
    if constexpr (VEC_IN) {
      // w_in % 4 == 0: every row is 16-byte aligned; w_eff rounded up stays inside the row
      for (uint32_t i = threadIdx.x; i < nc * w4; i += blockDim.x) {
        const uint32_t c = i / w4, q = i % w4;
        const float4 v = __ldg(reinterpret_cast<const float4*>(base + c * chan_stride) + q);
        float* t = tile + c * pitch + q * 4;
        t[0] = v.x; t[1] = v.y; t[2] = v.z; t[3] = v.w;
      }
    } else {
      for (uint32_t i = threadIdx.x; i < nc * w_eff; i += blockDim.x) {
        const uint32_t c = i / w_eff, col = i % w_eff;
        tile[c * pitch + col] = __ldg(base + c * chan_stride + col);
      }
    }
    __syncthreads();
    // thread -> (column, channel quad); 8 quads = 32 channels = one 128 B (fp32) segment
    const uint32_t nq = nc / 4;
    for (uint32_t i = threadIdx.x; i < w_eff * 8; i += blockDim.x) {
      const uint32_t col = i / 8, cq = i % 8;
      if (cq < nq) {
        const float* t = tile + cq * 4 * pitch + col;
        const float v0 = t[0], v1 = t[pitch], v2 = t[2 * pitch], v3 = t[3 * pitch];
        const uint64_t o = ((static_cast<uint64_t>(g) * w_eff + col) * h_f + fh) * c_in + c0 + cq * 4;
        if constexpr (BF16) {
          uint2 p;
          p.x = pack_bf16x2(v0, v1);
          p.y = pack_bf16x2(v2, v3);
          *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(dst) + o) = p;
        } else {
          *reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + o) = make_float4(v0, v1, v2, v3);
        }
      }
    }
    __syncthreads();
  }
}

// Narrow layers: work unit = (image, block of R output rows, 32-channel block).  The
// input rows those output rows read (span = (R-1)*s + Hf) are staged once per channel
// and every (output row, column, filter row) of the block is written from smem, so an
// input row is read from HBM/L2 once per unit instead of once per (g, fh).
template <bool BF16>
__global__ void __launch_bounds__(256) transform_cl_rows_kernel(const float* __restrict__ src, void* __restrict__ dst,
                                                                uint32_t c_in, uint32_t h_in, uint32_t w_in,
                                                                uint32_t h_out, uint32_t h_f, uint32_t stride,
                                                                uint32_t w_eff, uint32_t c_blocks, uint32_t rows,
                                                                uint32_t row_blocks, uint32_t cs,
                                                                uint32_t total_units, FastDiv fd_weff, FastDiv fd_hf) {
  extern __shared__ float tile[];  // [32][cs], row r at r*w_eff
  for (uint32_t u = blockIdx.x; u < total_units; u += gridDim.x) {
    const uint32_t cb = u % c_blocks;
    const uint32_t rb = (u / c_blocks) % row_blocks;
    const uint32_t img = u / (c_blocks * row_blocks);
    const uint32_t oh0 = rb * rows;
    const uint32_t nr = min(rows, h_out - oh0);
    const uint32_t span = (nr - 1) * stride + h_f;
    const uint32_t c0 = cb * 32;
    const uint32_t nc = min(32u, c_in - c0);
    const float* base = src + ((static_cast<uint64_t>(img) * c_in + c0) * h_in + oh0 * stride) * w_in;
    const uint64_t chan_stride = static_cast<uint64_t>(h_in) * w_in;
    const uint32_t per_c = span * w_eff;
    const FastDiv fd_perc(per_c);
    for (uint32_t i = threadIdx.x; i < nc * per_c; i += blockDim.x) {
      uint32_t c, rem, r, col;
      fd_perc.divmod(i, c, rem);
      fd_weff.divmod(rem, r, col);
      tile[c * cs + rem] = __ldg(base + c * chan_stride + r * w_in + col);
    }
    __syncthreads();
    const uint32_t nq = nc / 4;
    const uint32_t items = nr * w_eff * h_f * 8;
    for (uint32_t i = threadIdx.x; i < items; i += blockDim.x) {
      const uint32_t cq = i & 7;
      uint32_t rest, fh, col, ol;
      fd_hf.divmod(i >> 3, rest, fh);
      fd_weff.divmod(rest, ol, col);
      if (cq < nq) {
        const float* t = tile + cq * 4 * cs + (ol * stride + fh) * w_eff + col;
        const float v0 = t[0], v1 = t[cs], v2 = t[2 * cs], v3 = t[3 * cs];
        const uint64_t g = static_cast<uint64_t>(img) * h_out + oh0 + ol;
        const uint64_t o = ((g * w_eff + col) * h_f + fh) * c_in + c0 + cq * 4;
        if constexpr (BF16) {
          uint2 p;
          p.x = pack_bf16x2(v0, v1);
          p.y = pack_bf16x2(v2, v3);
          *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(dst) + o) = p;
        } else {
          *reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + o) = make_float4(v0, v1, v2, v3);
        }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- GEMM
struct ClArgs {
  float* __restrict__ out;  // (N, Co, Ho, Wo)
  uint32_t g_total;         // N*Ho
  uint32_t h_out, w_out, hw, co;
  uint32_t box_w, box_g;    // pixel tile = box_g rows x box_w columns
  uint32_t ow_tiles, g_tiles, co_tiles;
  uint32_t k_slabs;
};

template <bool BF16, int N, int STAGES>
__global__ void __launch_bounds__(256, 1)
    conv_tc_cl_kernel(const ClArgs a, const __grid_constant__ CUtensorMap tmap_a,
                      const __grid_constant__ CUtensorMap tmap_b) {
  constexpr uint32_t kABytes = kTileM * kRowBytes;
  constexpr uint32_t kBBytes = N * kRowBytes;
  constexpr uint32_t kStageBytes = kABytes + kBBytes;
  constexpr int kBK = BF16 ? 64 : 32;
  constexpr int kUK = BF16 ? 16 : 8;
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
  const uint32_t a_box_bytes = a.box_w * a.box_g * kRowBytes;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4);
    }
    fence_barrier_init();
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmap_a) : "memory");
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
  const uint32_t total_tiles = a.g_tiles * a.ow_tiles * a.co_tiles;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (uint32_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const uint32_t co_blk = t % a.co_tiles;
        const uint32_t pt = t / a.co_tiles;
        const uint32_t ow0 = (pt % a.ow_tiles) * a.box_w;
        const uint32_t g0 = (pt / a.ow_tiles) * a.box_g;
        for (uint32_t ks = 0; ks < a.k_slabs; ++ks) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * kStageBytes;
          mbar_arrive_expect_tx(&full_bar[stage], a_box_bytes + kBBytes);
          tma_load_3d(st, &tmap_a, &full_bar[stage], ks * kBK, ow0, g0);
          tma_load_2d(st + kABytes, &tmap_b, &full_bar[stage], ks * kBK, co_blk * N);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
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
          for (int kk = 0; kk < kBK / kUK; ++kk)
            mma<BF16>(tmem_d, smem_desc_sw128(abase + kk * 32), smem_desc_sw128(bbase + kk * 32), kIdesc,
                      (ks | kk) != 0);
          mma_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull_bar[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    const int quarter = warp % 4;
    const uint32_t r = quarter * 32 + lane;  // A row = TMEM lane
    const uint32_t rg = r / a.box_w, rw = r % a.box_w;
    uint32_t acc = 0, acc_phase = 0;
    for (uint32_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      const uint32_t co_blk = t % a.co_tiles;
      const uint32_t pt = t / a.co_tiles;
      const uint32_t ow = (pt % a.ow_tiles) * a.box_w + rw;
      const uint32_t g = (pt / a.ow_tiles) * a.box_g + rg;
      const bool valid = rg < a.box_g && ow < a.w_out && g < a.g_total;
      int64_t obase = 0;
      if (valid) {
        const uint32_t img = g / a.h_out, oh = g % a.h_out;
        obase = static_cast<int64_t>(img) * a.co * a.hw + static_cast<int64_t>(oh) * a.w_out + ow;
      }
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * N;
#pragma unroll
      for (int j0 = 0; j0 < N; j0 += 16) {
        uint32_t v[16];
        tmem_ld16(taddr + j0, v);
        const uint32_t m0 = co_blk * N + j0;
        if (valid) {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (m0 + q < a.co) a.out[obase + static_cast<int64_t>(m0 + q) * a.hw] = __uint_as_float(v[q]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

// B[m][k'] = F[m][c][fh][fw], k' = (fw*Hf + fh)*C + c, zero padded to Mp x Kp.
template <bool BF16>
__global__ void pack_filter_cl_kernel(const float* __restrict__ flt, void* __restrict__ packed, int M, int C, int h_f,
                                      int w_f, int Mp, int Kp) {
  const int K = C * h_f * w_f;
  const int64_t total = static_cast<int64_t>(Mp) * Kp;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i / Kp);
    const int kp = static_cast<int>(i % Kp);
    float v = 0.0f;
    if (m < M && kp < K) {
      const int c = kp % C, j = kp / C;
      const int fw = j / h_f, fh = j % h_f;
      v = flt[((static_cast<int64_t>(m) * C + c) * h_f + fh) * w_f + fw];
    }
    if constexpr (BF16) {
      reinterpret_cast<__nv_bfloat16*>(packed)[i] = __float2bfloat16_rn(v);
    } else {
      uint32_t r;
      asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(v));
      reinterpret_cast<uint32_t*>(packed)[i] = r;
    }
  }
}

static int pick_n_cl(int64_t co) {
  if (co <= 64) return 64;
  if (co <= 96) return 96;
  if (co <= 128) return 128;
  return 256;
}

template <bool BF16, int N, int STAGES>
static int launch_cl(ClArgs a, const void* win_cl, const void* packed, int64_t K, int64_t Kp, int64_t Mp,
                     int64_t c_in, int32_t h_f, int32_t stride, int64_t w_eff, cudaStream_t stream, const char** err) {
  constexpr int kBK = BF16 ? 64 : 32;
  auto enc = get_encode_fn();
  if (!enc) {
    *err = "conv_tc_cl: cuTensorMapEncodeTiled unavailable";
    return 2;
  }
  const cuuint64_t esz = BF16 ? 2 : 4;
  const CUtensorMapDataType dt = BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUtensorMap map_a, map_b;
  {
    // A: {k' < K, ow < Wo, g < N*Ho}; pixel stride s*Hf*C, row stride w_eff*Hf*C (windows overlap)
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), a.w_out, a.g_total};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(stride) * h_f * c_in * esz,
                             static_cast<cuuint64_t>(w_eff) * h_f * c_in * esz};
    cuuint32_t box[3] = {static_cast<cuuint32_t>(kBK), a.box_w, a.box_g};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&map_a, dt, 3, const_cast<void*>(win_cl), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      *err = "conv_tc_cl: window tensor map rejected (cuTensorMapEncodeTiled)";
      return 2;
    }
  }
  {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(Mp)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(Kp) * esz};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(N)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&map_b, dt, 2, const_cast<void*>(packed), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      *err = "conv_tc_cl: filter tensor map rejected (cuTensorMapEncodeTiled)";
      return 2;
    }
  }
  a.k_slabs = static_cast<uint32_t>(Kp / kBK);
  a.co_tiles = static_cast<uint32_t>(Mp / N);
  const size_t smem = static_cast<size_t>(STAGES) * (kTileM + N) * kRowBytes + 1024;
  auto kern = conv_tc_cl_kernel<BF16, N, STAGES>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 2;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t tiles = static_cast<uint64_t>(a.g_tiles) * a.ow_tiles * a.co_tiles;
  const uint32_t grid = tiles < static_cast<uint64_t>(sms) ? static_cast<uint32_t>(tiles) : static_cast<uint32_t>(sms);
  im2win_note_kernel("conv_tc_cl_kernel (TMA over the channels-innermost window tensor)");
  kern<<<grid, 256, smem, stream>>>(a, map_a, map_b);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 2;
  }
  return 0;
}

}  // namespace tc
}  // namespace im2win

int im2win_launch_transform_cl(const float* src, void* dst, int64_t n, int64_t c, int64_t h, int64_t w, int h_f,
                               int w_f, int stride, int bf16, cudaStream_t stream, const char** err) {
  const int64_t h_out = (h - h_f) / stride + 1;
  const int64_t w_out = (w - w_f) / stride + 1;
  const int64_t w_eff = (w_out - 1) * stride + w_f;
  const int64_t g_total = n * h_out;
  const int64_t c_blocks = (c + 31) / 32;
  const int64_t total = g_total * h_f * c_blocks;
  if (c % 4 != 0) {
    *err = "im2win_transform_cl: c must be a multiple of 4";
    return 1;
  }
  if ((reinterpret_cast<uintptr_t>(dst) & 15) != 0 || (reinterpret_cast<uintptr_t>(src) & 3) != 0) {
    *err = "im2win_transform_cl: dst must be 16-byte aligned and src 4-byte aligned";
    return 1;
  }
  if (total >= (1ll << 32) || n * c * h * w >= (1ll << 40)) {
    *err = "im2win_transform_cl: extents exceed the kernel's index range";
    return 1;
  }
  {
    // narrow rows: stage whole row blocks if 32 channels x span rows x w_eff fit in 48 KB
    const int64_t cap = 48 * 1024 / 4 / 32;  // floats per channel
    int64_t rows = 0;
    for (int64_t r = 1; r <= h_out; ++r) {
      const int64_t per_c = ((r - 1) * stride + h_f) * w_eff;
      if ((per_c + 31) / 32 * 32 + 1 > cap || r * w_eff * h_f * 32 > 32 * 1024) break;
      rows = r;
    }
    if (rows >= 2 || (rows == 1 && w_eff < 64)) {
      const int64_t span = (rows - 1) * stride + h_f;
      const uint32_t cs = static_cast<uint32_t>((span * w_eff + 31) / 32 * 32 + 1);
      const int64_t row_blocks = (h_out + rows - 1) / rows;
      const int64_t units = n * row_blocks * c_blocks;
      const size_t smem = static_cast<size_t>(32) * cs * 4;
      const uint32_t grid = static_cast<uint32_t>(units < 148 * 8 ? units : 148 * 8);
      if (bf16)
        im2win::tc::transform_cl_rows_kernel<true><<<grid, 256, smem, stream>>>(
            src, dst, static_cast<uint32_t>(c), static_cast<uint32_t>(h), static_cast<uint32_t>(w),
            static_cast<uint32_t>(h_out), h_f, stride, static_cast<uint32_t>(w_eff), static_cast<uint32_t>(c_blocks),
            static_cast<uint32_t>(rows), static_cast<uint32_t>(row_blocks), cs, static_cast<uint32_t>(units),
            im2win::FastDiv(static_cast<uint32_t>(w_eff)), im2win::FastDiv(static_cast<uint32_t>(h_f)));
      else
        im2win::tc::transform_cl_rows_kernel<false><<<grid, 256, smem, stream>>>(
            src, dst, static_cast<uint32_t>(c), static_cast<uint32_t>(h), static_cast<uint32_t>(w),
            static_cast<uint32_t>(h_out), h_f, stride, static_cast<uint32_t>(w_eff), static_cast<uint32_t>(c_blocks),
            static_cast<uint32_t>(rows), static_cast<uint32_t>(row_blocks), cs, static_cast<uint32_t>(units),
            im2win::FastDiv(static_cast<uint32_t>(w_eff)), im2win::FastDiv(static_cast<uint32_t>(h_f)));
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) {
        *err = cudaGetErrorString(e);
        return 2;
      }
      return 0;
    }
  }
  const uint32_t w4 = static_cast<uint32_t>((w_eff + 3) / 4);
  const uint32_t pitch = (w4 * 4 + 31) / 32 * 32 + 1;
  const size_t smem = static_cast<size_t>(32) * pitch * 4;
  const uint32_t grid = static_cast<uint32_t>(total < 148 * 8 ? total : 148 * 8);
  const bool vec = (w % 4 == 0) && (reinterpret_cast<uintptr_t>(src) % 16 == 0);
#define IM2WIN_TCL(BF, V)                                                                                         \
  {                                                                                                               \
    auto k = im2win::tc::transform_cl_kernel<BF, V>;                                                              \
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)); \
    k<<<grid, 256, smem, stream>>>(src, dst, static_cast<uint32_t>(c), static_cast<uint32_t>(h),                  \
                                   static_cast<uint32_t>(w), static_cast<uint32_t>(h_out), h_f, stride,           \
                                   static_cast<uint32_t>(w_eff), static_cast<uint32_t>(c_blocks), pitch,          \
                                   static_cast<uint32_t>(total));                                                 \
  }
  if (bf16) {
    if (vec) IM2WIN_TCL(true, true) else IM2WIN_TCL(true, false)
  } else {
    if (vec) IM2WIN_TCL(false, true) else IM2WIN_TCL(false, false)
  }
#undef IM2WIN_TCL
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 2;
  }
  return 0;
}

size_t im2win_tc_cl_workspace_bytes(int64_t c_out, int64_t K) {
  const int64_t Mp = (c_out + 255) / 256 * 256 + 256;
  const int64_t Kp = (K + 63) / 64 * 64;
  return static_cast<size_t>(Mp * Kp) * 4 + 1024;
}

int im2win_launch_conv_tc_cl(const void* win_cl, const float* flt, float* out, void* workspace, int64_t n,
                             int64_t c_in, int64_t c_out, int64_t h_out, int64_t w_out, int h_f, int w_f, int stride,
                             int bf16, cudaStream_t stream, const char** err) {
  using namespace im2win::tc;
  const int64_t esz = bf16 ? 2 : 4;
  if ((c_in * esz) % 16 != 0) {
    *err = "im2win_conv_cl: c_in * element size must be a multiple of 16 bytes";
    return 1;
  }
  const int64_t K = c_in * h_f * w_f;
  const int64_t w_eff = (w_out - 1) * stride + w_f;
  const int N = pick_n_cl(c_out);
  const int bk = bf16 ? 64 : 32;
  const int64_t Kp = (K + bk - 1) / bk * bk;
  const int64_t Mp = (c_out + N - 1) / N * N;
  ClArgs a{};
  a.out = out;
  a.g_total = static_cast<uint32_t>(n * h_out);
  a.h_out = static_cast<uint32_t>(h_out);
  a.w_out = static_cast<uint32_t>(w_out);
  a.hw = static_cast<uint32_t>(h_out * w_out);
  a.co = static_cast<uint32_t>(c_out);
  if (w_out <= kTileM) {
    a.box_w = static_cast<uint32_t>(w_out);
    a.box_g = static_cast<uint32_t>(kTileM / w_out);
  } else {
    const int64_t parts = (w_out + kTileM - 1) / kTileM;
    a.box_w = static_cast<uint32_t>((w_out + parts - 1) / parts);
    a.box_g = 1;
  }
  if (a.box_g > 256) a.box_g = 256;
  a.ow_tiles = (a.w_out + a.box_w - 1) / a.box_w;
  a.g_tiles = (a.g_total + a.box_g - 1) / a.box_g;
  if (bf16)
    pack_filter_cl_kernel<true><<<256, 256, 0, stream>>>(flt, workspace, static_cast<int>(c_out), static_cast<int>(c_in),
                                                         h_f, w_f, static_cast<int>(Mp), static_cast<int>(Kp));
  else
    pack_filter_cl_kernel<false><<<256, 256, 0, stream>>>(flt, workspace, static_cast<int>(c_out), static_cast<int>(c_in),
                                                          h_f, w_f, static_cast<int>(Mp), static_cast<int>(Kp));
#define IM2WIN_CL(BF, NN, ST) \
  return launch_cl<BF, NN, ST>(a, win_cl, workspace, K, Kp, Mp, c_in, h_f, stride, w_eff, stream, err)
  if (bf16) {
    switch (N) {
      case 64: IM2WIN_CL(true, 64, 8);
      case 96: IM2WIN_CL(true, 96, 6);
      case 128: IM2WIN_CL(true, 128, 6);
      default: IM2WIN_CL(true, 256, 4);
    }
  } else {
    switch (N) {
      case 64: IM2WIN_CL(false, 64, 8);
      case 96: IM2WIN_CL(false, 96, 6);
      case 128: IM2WIN_CL(false, 128, 6);
      default: IM2WIN_CL(false, 256, 4);
    }
  }
#undef IM2WIN_CL
}
