// Window-shift tensor-core convolution for stride-1 layers (the im2win reuse in hardware).
//
// im2win stores windows so that consecutive output columns' windows overlap
// (layouts.py:187-199: window ow is the slice [ow*s*Hf, ow*s*Hf + Hf*Wf) of the row).
// For stride 1 the A-tile rows of filter column fw are the rows of filter column 0
// shifted by fw: A_fw[pixel r][c] = A_0[pixel r + fw][c].  So one TMA box per
// (fh, channel chunk) loads R x P input pixels (P = box_w + Wf - 1 columns per output
// row) from the channels-last input, and the Wf MMAs of that K-slab read it through
// descriptors whose start address is advanced by fw rows (fw * 128 B).  A is fetched
// once per (fh, chunk) instead of once per (fh, fw, chunk): L2->SM traffic for A drops
// by Wf.  D rows whose column position is >= box_w are padding and are not stored.
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "tc_common.cuh"

namespace im2win {
namespace tc {

struct ShiftArgs {
  float* __restrict__ out;
  uint32_t n_img, h_out, w_out, hw, co;
  uint32_t box_w, pitch, rows, box_n;  // P = pitch = box_w + Wf - 1; R = rows output rows; box_n images
  uint32_t ow_tiles, oh_tiles, n_tiles, co_tiles;
  uint32_t c_slabs, w_f, k_slabs;      // k_slabs = Hf * c_slabs; Kc = c_slabs * BK
};

constexpr int kARows = 136;  // 128 MMA rows + up to 8 rows of shift (Wf <= 9)

IM2WIN_DEVICE uint64_t smem_desc_sw128_off(uint32_t addr) {
  uint64_t d = smem_desc_sw128(addr);
  d |= static_cast<uint64_t>((addr >> 7) & 7) << 49;  // matrix base offset: row phase inside the 1024 B atom
  return d;
}

template <bool BF16, int N, int STAGES, int WF, bool RB>
__global__ void __launch_bounds__(kTcThreadsFeed, 1)
    conv_tc_shift_kernel(const ShiftArgs a, const __grid_constant__ CUtensorMap tmap_a,
                         const __grid_constant__ CUtensorMap tmap_b, const NhwcFeed feed) {
  constexpr uint32_t kABytes = kARows * kRowBytes;  // 17 KB (multiple of 1024)
  constexpr uint32_t kBBytes = RB ? 0 : WF * N * kRowBytes;  // RB: filter resident, not staged
  constexpr uint32_t kStageBytes = kABytes + kBBytes;
  constexpr int kBK = BF16 ? 64 : 32;
  constexpr int kUK = BF16 ? 16 : 8;
  constexpr uint32_t kTmemCols = (2 * N <= 128) ? 128 : (2 * N <= 256 ? 256 : 512);
  constexpr uint32_t kIdesc = instr_desc<BF16, N>();
  static_assert(kABytes % 1024 == 0, "A stage must keep 1024 B alignment");

  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2];
  __shared__ __align__(8) uint64_t tempty_bar[2];
  __shared__ __align__(8) uint64_t bres_bar;
  __shared__ uint32_t tmem_base_sh;

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t loaded_rows = a.pitch * a.rows * a.box_n;
  const uint32_t a_box_bytes = loaded_rows * kRowBytes;
  // RB: the whole packed filter (k_slabs x Wf tiles of N x 128 B) sits in front of the A stages
  const uint32_t rb_bytes = RB ? a.k_slabs * WF * N * kRowBytes : 0;
  uint8_t* stages = smem + rb_bytes;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      if (s == 0) mbar_init(&bres_bar, 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], kEpiWarps);
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
  // rows past the TMA box feed only padding D rows, but keep them finite
  for (uint32_t i = threadIdx.x; i < STAGES * kABytes / 16; i += blockDim.x) {
    const uint32_t s = i / (kABytes / 16), off = i % (kABytes / 16);
    reinterpret_cast<uint4*>(stages + s * kStageBytes)[off] = make_uint4(0, 0, 0, 0);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;
  const uint32_t total_tiles = a.n_tiles * a.oh_tiles * a.ow_tiles * a.co_tiles;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      if constexpr (RB) {  // requires co_tiles == 1 (host-checked)
        mbar_arrive_expect_tx(&bres_bar, rb_bytes);
        for (uint32_t ks = 0; ks < a.k_slabs; ++ks)
          for (int fw = 0; fw < WF; ++fw)
            tma_load_2d(smem + (ks * WF + fw) * N * kRowBytes, &tmap_b, &bres_bar,
                        ((ks / a.c_slabs) * WF + fw) * a.c_slabs * kBK + (ks % a.c_slabs) * kBK, 0);
      }
      uint32_t conf_lo = 1, conf_hi = 0;
      for (uint32_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const uint32_t co_blk = t % a.co_tiles;
        uint32_t pt = t / a.co_tiles;
        const uint32_t ow0 = (pt % a.ow_tiles) * a.box_w;
        pt /= a.ow_tiles;
        const uint32_t oh0 = (pt % a.oh_tiles) * a.rows;
        const uint32_t n0 = (pt / a.oh_tiles) * a.box_n;
        nhwc_feed_wait(feed, n0, n0 + a.box_n - 1, conf_lo, conf_hi);
        for (uint32_t ks = 0; ks < a.k_slabs; ++ks) {
          const uint32_t fh = ks / a.c_slabs;
          const uint32_t c0 = (ks % a.c_slabs) * kBK;
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = stages + stage * kStageBytes;
          mbar_arrive_expect_tx(&full_bar[stage], a_box_bytes + kBBytes);
          // A: {c, input col, input row, image} box {BK, P, R, box_n} at (c0, ow0, oh0 + fh, n0)
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
              "%6}], [%2];\n" ::"r"(smem_u32(st)),
              "l"(&tmap_a), "r"(smem_u32(&full_bar[stage])), "r"(c0), "r"(ow0), "r"(oh0 + fh), "r"(n0)
              : "memory");
          if constexpr (!RB)
#pragma unroll
            for (int fw = 0; fw < WF; ++fw)
              tma_load_2d(st + kABytes + fw * N * kRowBytes, &tmap_b, &full_bar[stage],
                        (fh * WF + fw) * a.c_slabs * kBK + c0, co_blk * N);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      if constexpr (RB) mbar_wait(&bres_bar, 0);
      for (uint32_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * N;
        for (uint32_t ks = 0; ks < a.k_slabs; ++ks) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t abase = smem_u32(stages + stage * kStageBytes);
          const uint32_t bbase = RB ? smem_u32(smem) + ks * WF * N * kRowBytes : abase + kABytes;
#pragma unroll
          for (int fw = 0; fw < WF; ++fw) {
#pragma unroll
            for (int kk = 0; kk < kBK / kUK; ++kk) {
              const uint32_t aaddr = abase + fw * kRowBytes + kk * 32;
              const uint64_t ad = smem_desc_sw128(aaddr);
              mma<BF16>(tmem_d, ad, smem_desc_sw128(bbase + fw * N * kRowBytes + kk * 32), kIdesc,
                        (ks | fw | kk) != 0);
            }
          }
          mma_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull_bar[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4 + kEpiWarps) {
    if (feed.src)
      nhwc_feed_run<BF16>(feed, lane, blockIdx.x * kFeedWarps + (warp - 4 - kEpiWarps), gridDim.x * kFeedWarps);
  } else if (warp >= 4) {
    // kEpiWarps epilogue warps: warp w reads TMEM lane quarter w % 4 and column half (w - 4) / 4
    const int quarter = warp % 4;
    const int j_lo = ((warp - 4) / 4) * (N / 2);
    const uint32_t r = quarter * 32 + lane;
    const uint32_t per_img = a.pitch * a.rows;
    const uint32_t r_n = r / per_img, r_rem = r % per_img;
    const uint32_t r_h = r_rem / a.pitch, r_w = r_rem % a.pitch;
    uint32_t acc = 0, acc_phase = 0;
    for (uint32_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      const uint32_t co_blk = t % a.co_tiles;
      uint32_t pt = t / a.co_tiles;
      const uint32_t ow = (pt % a.ow_tiles) * a.box_w + r_w;
      pt /= a.ow_tiles;
      const uint32_t oh = (pt % a.oh_tiles) * a.rows + r_h;
      const uint32_t img = (pt / a.oh_tiles) * a.box_n + r_n;
      const bool valid = r < loaded_rows && r_w < a.box_w && ow < a.w_out && oh < a.h_out && img < a.n_img;
      const int64_t obase = valid ? static_cast<int64_t>(img) * a.co * a.hw + static_cast<int64_t>(oh) * a.w_out + ow : 0;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * N;
#pragma unroll
      for (int jj = 0; jj < N / 2; jj += 16) {
        const int j0 = j_lo + jj;
        uint32_t v[16];
        tmem_ld16(taddr + j0, v);
        const uint32_t m0 = co_blk * N + j0;
        if (valid) {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (m0 + q < a.co) st_out(a.out + obase + static_cast<int64_t>(m0 + q) * a.hw, __uint_as_float(v[q]));
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

// B[m][(fh*Wf + fw)*Kc + c] = F[m][c][fh][fw] (zero for c >= C).
template <bool BF16>
__global__ void pack_filter_shift_kernel(const float* __restrict__ flt, void* __restrict__ packed, int M, int C,
                                         int h_f, int w_f, int Mp, int Kc) {
  const int64_t Kp = static_cast<int64_t>(h_f) * w_f * Kc;
  const int64_t total = Mp * Kp;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i / Kp);
    const int64_t kp = i % Kp;
    const int tap = static_cast<int>(kp / Kc), c = static_cast<int>(kp % Kc);
    const int fh = tap / w_f, fw = tap % w_f;
    float v = 0.0f;
    if (m < M && c < C) v = flt[((static_cast<int64_t>(m) * C + c) * h_f + fh) * w_f + fw];
    if constexpr (BF16) {
      reinterpret_cast<__nv_bfloat16*>(packed)[i] = __float2bfloat16_rn(v);
    } else {
      uint32_t r;
      asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(v));
      reinterpret_cast<uint32_t*>(packed)[i] = r;
    }
  }
}

// Tile shape for the shift kernel; returns the fraction of the 128 MMA rows that are real outputs.
inline double shift_tile(int64_t n, int64_t h_out, int64_t w_out, int w_f, ShiftArgs& a) {
  const int64_t max_w = kTileM - (w_f - 1);
  if (w_out <= max_w) {
    a.box_w = static_cast<uint32_t>(w_out);
    a.pitch = static_cast<uint32_t>(w_out + w_f - 1);
    const int64_t rmax = std::max<int64_t>(1, kTileM / a.pitch);
    a.rows = static_cast<uint32_t>(std::min<int64_t>(h_out, rmax));
    a.box_n = a.rows == h_out ? static_cast<uint32_t>(std::max<int64_t>(1, std::min<int64_t>(n, kTileM / (a.pitch * h_out))))
                              : 1u;
  } else {
    const int64_t parts = (w_out + max_w - 1) / max_w;
    a.box_w = static_cast<uint32_t>((w_out + parts - 1) / parts);
    a.pitch = a.box_w + w_f - 1;
    a.rows = 1;
    a.box_n = 1;
  }
  return static_cast<double>(a.box_w) * a.rows * a.box_n / kTileM;
}

template <bool BF16, int N, int STAGES, int WF, bool RB>
static int launch_shift(ShiftArgs a, const void* x_cl, const void* packed, int64_t c_in, int64_t h, int64_t w,
                        int64_t Mp, int64_t Kp, const NhwcFeed& feed, cudaStream_t stream, const char** err) {
  constexpr int kBK = BF16 ? 64 : 32;
  auto enc = get_encode_fn();
  if (!enc) {
    *err = "conv_tc_shift: cuTensorMapEncodeTiled unavailable";
    return 2;
  }
  const cuuint64_t esz = BF16 ? 2 : 4;
  const CUtensorMapDataType dt = BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUtensorMap map_a, map_b;
  {
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(c_in), static_cast<cuuint64_t>(w), static_cast<cuuint64_t>(h),
                          a.n_img};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(c_in) * esz, static_cast<cuuint64_t>(w) * c_in * esz,
                             static_cast<cuuint64_t>(h) * w * c_in * esz};
    cuuint32_t box[4] = {static_cast<cuuint32_t>(kBK), a.pitch, a.rows, a.box_n};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(&map_a, dt, 4, const_cast<void*>(x_cl), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      *err = "conv_tc_shift: input tensor map rejected (cuTensorMapEncodeTiled)";
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
      *err = "conv_tc_shift: filter tensor map rejected (cuTensorMapEncodeTiled)";
      return 2;
    }
  }
  a.co_tiles = static_cast<uint32_t>(Mp / N);
  const size_t rb = RB ? static_cast<size_t>(a.k_slabs) * WF * N * kRowBytes : 0;
  const size_t smem = rb + static_cast<size_t>(STAGES) * (kARows + (RB ? 0 : WF * N)) * kRowBytes + 1024;
  // Measured on B200: the SW128 swizzle phase follows the absolute smem address, so the
  // row-shifted start address needs no descriptor base offset.
  auto kern = conv_tc_shift_kernel<BF16, N, STAGES, WF, RB>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 2;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t tiles = static_cast<uint64_t>(a.n_tiles) * a.oh_tiles * a.ow_tiles * a.co_tiles;
  const uint32_t grid = tiles < static_cast<uint64_t>(sms) ? static_cast<uint32_t>(tiles) : static_cast<uint32_t>(sms);
  im2win_note_kernel(RB ? "conv_tc_shift_kernel (window shift, filter resident)" : "conv_tc_shift_kernel (window shift)");
  e = launch_tc_kernel(kern, grid, smem, stream, feed.src != nullptr, 1, a, map_a, map_b, feed_for(feed, grid, tiles));
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 2;
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 2;
  }
  return 0;
}

}  // namespace tc
}  // namespace im2win

// Returns 1 and launches when the shift kernel applies (stride 1, Wf in {3, 5}, tile
// utilisation not worse than the generic fused tile), 0 when the caller should use the
// generic fused kernel, <0 on error.
int im2win_try_conv_tc_shift(const void* x_cl, const float* flt, float* out, void* workspace, int64_t n, int64_t c_in,
                             int64_t c_pad, int64_t h, int64_t w, int64_t c_out, int h_f, int w_f, int stride, int bf16,
                             double fused_util, const im2win::tc::NhwcFeed& feed, cudaStream_t stream,
                             const char** err) {
  using namespace im2win::tc;
  if (stride != 1 || (w_f != 3 && w_f != 5)) return 0;
  const char* env = getenv("IM2WIN_SHIFT");
  const int mode = env ? atoi(env) : 1;  // 0 off, 1 auto, 2 wherever legal
  if (mode == 0) return 0;
  // few channels (conv7, C = 3): a tap's A row is mostly channel padding; measured slower than
  // the generic kernel (tools/tc_kernels.py conv7: 28 vs 33 TF)
  if (mode == 1 && c_in < 16) return 0;
  const int64_t h_out = h - h_f + 1, w_out = w - w_f + 1;
  ShiftArgs a{};
  a.out = out;
  a.n_img = static_cast<uint32_t>(n);
  a.h_out = static_cast<uint32_t>(h_out);
  a.w_out = static_cast<uint32_t>(w_out);
  a.hw = static_cast<uint32_t>(h_out * w_out);
  a.co = static_cast<uint32_t>(c_out);
  const double util = shift_tile(n, h_out, w_out, w_f, a);
  if (util + 1e-9 < fused_util * 0.9) return 0;
  // B per stage = Wf * N * 128 B must leave room for >= 3 stages: N <= 128 for Wf=3, N = 64 for Wf=5.
  // Wider Co would need a Co split (A re-read per split), measured slower than the generic kernel.
  if (c_out > 128 || (w_f == 5 && c_out > 64)) return 0;
  const int N = c_out <= 64 ? 64 : 128;
  const int bk = bf16 ? 64 : 32;
  const int64_t c_slabs = (c_in + bk - 1) / bk;
  const int64_t Kc = c_slabs * bk;
  const int64_t Kp = static_cast<int64_t>(h_f) * w_f * Kc;
  const int64_t Mp = (c_out + N - 1) / N * N;
  a.ow_tiles = (a.w_out + a.box_w - 1) / a.box_w;
  a.oh_tiles = (a.h_out + a.rows - 1) / a.rows;
  a.n_tiles = (a.n_img + a.box_n - 1) / a.box_n;
  a.c_slabs = static_cast<uint32_t>(c_slabs);
  a.w_f = static_cast<uint32_t>(w_f);
  a.k_slabs = static_cast<uint32_t>(h_f * c_slabs);
  if (bf16)
    pack_filter_shift_kernel<true><<<256, 256, 0, stream>>>(flt, workspace, static_cast<int>(c_out),
                                                            static_cast<int>(c_in), h_f, w_f, static_cast<int>(Mp),
                                                            static_cast<int>(Kc));
  else
    pack_filter_shift_kernel<false><<<256, 256, 0, stream>>>(flt, workspace, static_cast<int>(c_out),
                                                             static_cast<int>(c_in), h_f, w_f, static_cast<int>(Mp),
                                                             static_cast<int>(Kc));
  int rc;
  // Filter-resident mode: when the packed filter fits next to 4 A stages it is loaded
  // once per CTA (one Co tile) and only window tiles stream through the ring.
  const size_t rb_bytes = static_cast<size_t>(a.k_slabs) * w_f * N * kRowBytes;
  const bool rb = Mp == N && rb_bytes + 4 * kARows * kRowBytes + 1024 <= 227 * 1024 &&
                  !(getenv("IM2WIN_SHIFT_RB") && atoi(getenv("IM2WIN_SHIFT_RB")) == 0);
#define IM2WIN_SH(BF, NN, ST, WFF, RBB) \
  rc = launch_shift<BF, NN, ST, WFF, RBB>(a, x_cl, workspace, c_pad, h, w, Mp, Kp, feed, stream, err)
  if (w_f == 3) {
    if (bf16) {
      if (N == 64) { if (rb) IM2WIN_SH(true, 64, 4, 3, true); else IM2WIN_SH(true, 64, 5, 3, false); }
      else { if (rb) IM2WIN_SH(true, 128, 4, 3, true); else IM2WIN_SH(true, 128, 3, 3, false); }
    } else {
      if (N == 64) { if (rb) IM2WIN_SH(false, 64, 4, 3, true); else IM2WIN_SH(false, 64, 5, 3, false); }
      else { if (rb) IM2WIN_SH(false, 128, 4, 3, true); else IM2WIN_SH(false, 128, 3, 3, false); }
    }
  } else {
    if (bf16) { if (rb) IM2WIN_SH(true, 64, 4, 5, true); else IM2WIN_SH(true, 64, 3, 5, false); }
    else { if (rb) IM2WIN_SH(false, 64, 4, 5, true); else IM2WIN_SH(false, 64, 3, 5, false); }
  }
#undef IM2WIN_SH
  return rc == 0 ? 1 : -rc;
}
