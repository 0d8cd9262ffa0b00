// Fused ("implicit") im2win tensor-core convolution: window tiles are built by TMA
// straight from a channels-last copy of the input, so Ĩ is never materialised.
//
// With Xcl[n][h][w][c] (NHWC), the im2win window row of filter row fh for output pixel
// (n, oh, ow) is ONE contiguous run of Wf*C elements, Xcl[n][oh*s+fh][ow*s .. ow*s+Wf-1][:],
// i.e. exactly the channels-last window row of the im2win layout (layouts.py:73-83 stores
// the same Hf rows per output row; here the TMA engine gathers them per tile).  The GEMM
// operand is therefore the strided 5-D view
//     A[(n, oh, ow)][(fh, j)] = Xcl + n*H*W*C + (oh*s + fh)*W*C + ow*s*C + j,  j < Wf*C
// {j, fh, ow, oh, n} with strides {1, W*C, s*C, s*W*C, H*W*C} elements, which one
// cp.async.bulk.tensor.5d per K-slab streams into the 128-byte-swizzled K-major smem
// tile tcgen05.mma reads.  K-slabs run over (fh, 32/64-wide chunks of j); the pixel
// tile is a box of box_w x box_h x box_n output pixels (<= 128 = UMMA M).
// HBM traffic: read X, write Xcl (1x input), the conv reads Xcl (L2 absorbs the
// Hf*Wf/s^2 window overlap) -- versus writing and re-reading the 2-4x larger Ĩ.
#include <stddef.h>
#include <algorithm>
#include <cstdlib>
#include <stdint.h>

#include "tc_common.cuh"

namespace im2win {
namespace tc {

// Destination pixel index of source pixel p (row-major in an h x w image) in a
// channels-last copy whose spatial extent is zero-padded by `pad` on every side.
struct PadMap {
  uint32_t pad, wp;   // wp = w + 2*pad
  uint64_t img_px;    // (h + 2*pad) * wp pixels per image
  FastDiv fd_w;
  IM2WIN_DEVICE uint64_t pixel(uint64_t img, uint32_t p) const {
    if (pad == 0) return img * img_px + p;
    uint32_t y, x;
    fd_w.divmod(p, y, x);
    return img * img_px + static_cast<uint64_t>(y + pad) * wp + x + pad;
  }
};

// NCHW float32 -> NHWC (float32 or bf16) with the channel pitch padded to c_pad
// (a 16-byte multiple, zero filled): per image a [C][H*W] -> [H*W][c_pad] transpose.
template <bool BF16>
__global__ void __launch_bounds__(256) nchw_to_nhwc_kernel(const float* __restrict__ src, void* __restrict__ dst,
                                                           uint32_t c_in, uint32_t c_pad, uint32_t hw,
                                                           uint32_t hw_tiles, uint32_t c_tiles, uint32_t total,
                                                           const PadMap pm) {
  __shared__ float tile[32][33];
  const uint32_t tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  for (uint32_t b = blockIdx.x; b < total; b += gridDim.x) {
    const uint32_t ct = b % c_tiles;
    const uint32_t pt = (b / c_tiles) % hw_tiles;
    const uint32_t img = b / (c_tiles * hw_tiles);
    const uint32_t c0 = ct * 32, p0 = pt * 32;
    const float* s = src + static_cast<uint64_t>(img) * c_in * hw;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t c = c0 + ty + 8 * j, p = p0 + tx;
      tile[ty + 8 * j][tx] = (c < c_in && p < hw) ? __ldg(s + static_cast<uint64_t>(c) * hw + p) : 0.0f;
    }
    __syncthreads();
    // write: 8 threads per pixel, 4 channels each (16 B fp32 / 8 B bf16)
    const uint32_t pl = threadIdx.x / 8, cq = threadIdx.x % 8;
    const uint32_t p = p0 + pl, c = c0 + cq * 4;
    if (p < hw && c < c_pad) {
      const float v0 = tile[cq * 4][pl], v1 = tile[cq * 4 + 1][pl], v2 = tile[cq * 4 + 2][pl], v3 = tile[cq * 4 + 3][pl];
      const uint64_t o = pm.pixel(img, p) * c_pad + c;
      if constexpr (BF16) {
        uint2 q;
        q.x = pack_bf16x2(v0, v1);
        q.y = pack_bf16x2(v2, v3);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(dst) + o) = q;
      } else {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + o) = make_float4(v0, v1, v2, v3);
      }
    }
    __syncthreads();
  }
}

// Small-image variant (H*W <= 256 and not a multiple of 4, e.g. 7x7: conv12): a CTA moves a
// 32-channel slab of one image, which is one contiguous run of 32*H*W floats -- loaded with
// 16-byte loads when the image is 16-byte aligned -- transposed in smem (odd row pitch) and
// written as whole 128-byte (fp32) / 64-byte (bf16) pixel rows.  The 32x32 generic kernel moves
// such images at ~3.3 TB/s: half of its second pixel tile is empty and its loads are scalar.
template <bool BF16>
__global__ void __launch_bounds__(128) nchw_to_nhwc_block_kernel(const float* __restrict__ src, void* __restrict__ dst,
                                                                 uint32_t c_in, uint32_t c_pad, uint32_t hw,
                                                                 uint32_t c_tiles, uint32_t total, uint32_t vec,
                                                                 const PadMap pm) {
  extern __shared__ float tile[];  // [32][pitch]: small, so many CTAs (and their loads) per SM
  const uint32_t pitch = hw | 1u;
  constexpr uint32_t G = BF16 ? 8 : 4;  // channels per 16-byte store
  for (uint32_t b = blockIdx.x; b < total; b += gridDim.x) {
    const uint32_t ct = b % c_tiles, img = b / c_tiles;
    const uint32_t c0 = ct * 32;
    const uint32_t nc = min(32u, c_in - c0);
    const float* s = src + (static_cast<uint64_t>(img) * c_in + c0) * hw;
    const uint32_t cnt = nc * hw;
    if (vec) {
      for (uint32_t q = threadIdx.x; q < cnt / 4; q += blockDim.x) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(s) + q);
        const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t f = 4 * q + j, c = f / hw;
          tile[c * pitch + (f - c * hw)] = e[j];
        }
      }
    } else {
      for (uint32_t f = threadIdx.x; f < cnt; f += blockDim.x) {
        const uint32_t c = f / hw;
        tile[c * pitch + (f - c * hw)] = __ldg(s + f);
      }
    }
    __syncthreads();
    // write: 32/G threads per pixel, G channels each; channels >= c_in (pitch padding) are zeros
    const uint32_t per = 32 / G;
    const uint32_t groups = min(per, (c_pad - c0 + G - 1) / G);
    for (uint32_t i = threadIdx.x; i < hw * per; i += blockDim.x) {
      const uint32_t p = i / per, g = i % per;
      if (g >= groups) continue;
      float v[G];
#pragma unroll
      for (uint32_t j = 0; j < G; ++j) {
        const uint32_t c = g * G + j;
        v[j] = c < nc ? tile[c * pitch + p] : 0.0f;
      }
      const uint64_t o = pm.pixel(img, p) * c_pad + c0 + g * G;
      if constexpr (BF16) {
        uint4 q;
        q.x = pack_bf16x2(v[0], v[1]);
        q.y = pack_bf16x2(v[2], v[3]);
        q.z = pack_bf16x2(v[4], v[5]);
        q.w = pack_bf16x2(v[6], v[7]);
        __stcs(reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(dst) + o), q);
      } else {
        __stcs(reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + o), make_float4(v[0], v[1], v[2], v[3]));
      }
    }
    __syncthreads();
  }
}

// Wide-tile variant (c_pad > 8, Ho*Wo % 4 == 0): a CTA moves a 64-channel x 64-pixel
// tile per iteration -- four 16-byte loads per thread in flight, a padded smem
// transpose (row pitch 65 floats), and 16-byte channels-last stores (4 fp32 or 8 bf16
// channels per store, the channel pitch is a multiple of that granule).
template <bool BF16>
__global__ void __launch_bounds__(256) nchw_to_nhwc_wide_kernel(const float* __restrict__ src, void* __restrict__ dst,
                                                                uint32_t c_in, uint32_t c_pad, uint32_t hw,
                                                                uint32_t hw_tiles, uint32_t c_tiles, uint32_t total,
                                                                const PadMap pm) {
  __shared__ float tile[64][65];
  const uint32_t t = threadIdx.x;
  for (uint32_t b = blockIdx.x; b < total; b += gridDim.x) {
    const uint32_t ct = b % c_tiles;
    const uint32_t pt = (b / c_tiles) % hw_tiles;
    const uint32_t img = b / (c_tiles * hw_tiles);
    const uint32_t c0 = ct * 64, p0 = pt * 64;
    const float* s = src + static_cast<uint64_t>(img) * c_in * hw;
    // load: thread t covers pixels p0 + 4*(t%16) .. +3 of channels c0 + t/16 + 16*j
    float4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t c = c0 + t / 16 + 16 * j, p = p0 + 4 * (t % 16);
      v[j] = (c < c_in && p < hw) ? __ldcs(reinterpret_cast<const float4*>(s + static_cast<uint64_t>(c) * hw + p))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float* row = &tile[t / 16 + 16 * j][4 * (t % 16)];
      row[0] = v[j].x; row[1] = v[j].y; row[2] = v[j].z; row[3] = v[j].w;
    }
    __syncthreads();
    // store: kPer threads per pixel, one 16-byte granule (G channels) each, granule fastest:
    // a warp instruction writes contiguous pixel rows (512 B), no partial sectors
    constexpr uint32_t G = BF16 ? 8 : 4;
    constexpr uint32_t kPer = 64 / G;         // threads per pixel
    constexpr uint32_t kPass = 256 / kPer;    // pixels per pass
    const uint32_t cq = t % kPer;
    const uint32_t cl = cq * G, c = c0 + cl;
#pragma unroll
    for (uint32_t pp = 0; pp < 64; pp += kPass) {
      const uint32_t pl = pp + t / kPer;
      const uint32_t p = p0 + pl;
      if (p < hw && c < c_pad) {
        const uint64_t o = pm.pixel(img, p) * c_pad;
        if constexpr (BF16) {
          uint4 q;
          q.x = pack_bf16x2(tile[cl][pl], tile[cl + 1][pl]);
          q.y = pack_bf16x2(tile[cl + 2][pl], tile[cl + 3][pl]);
          q.z = pack_bf16x2(tile[cl + 4][pl], tile[cl + 5][pl]);
          q.w = pack_bf16x2(tile[cl + 6][pl], tile[cl + 7][pl]);
          __stcs(reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(dst) + o + c), q);
        } else {
          __stcs(reinterpret_cast<float4*>(reinterpret_cast<float*>(dst) + o + c),
                 make_float4(tile[cl][pl], tile[cl + 1][pl], tile[cl + 2][pl], tile[cl + 3][pl]));
        }
      }
    }
    __syncthreads();
  }
}

// Few channels (c_pad <= 8, e.g. the RGB input layers): one thread per pixel reads its
// C values (coalesced along the pixel axis) and writes the padded pixel with one
// 16/32-byte store; the 32-channel smem transpose would leave most of its tile empty.
template <bool BF16>
__global__ void __launch_bounds__(256) nchw_to_nhwc_small_kernel(const float* __restrict__ src, void* __restrict__ dst,
                                                                 uint32_t c_in, uint32_t c_pad, uint64_t hw,
                                                                 uint64_t total, const PadMap pm) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t img = i / hw, p = i % hw;
    const float* s = src + img * c_in * hw + p;
    const uint64_t od = pm.pixel(img, static_cast<uint32_t>(p));
    float v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = (static_cast<uint32_t>(c) < c_in) ? __ldg(s + c * hw) : 0.0f;
    if constexpr (BF16) {
      // c_pad == 8 for bf16 (16-byte pitch)
      uint4 q;
      q.x = pack_bf16x2(v[0], v[1]);
      q.y = pack_bf16x2(v[2], v[3]);
      q.z = pack_bf16x2(v[4], v[5]);
      q.w = pack_bf16x2(v[6], v[7]);
      reinterpret_cast<uint4*>(dst)[od] = q;
    } else {
      float4* d = reinterpret_cast<float4*>(dst) + od * (c_pad / 4);
      d[0] = make_float4(v[0], v[1], v[2], v[3]);
      if (c_pad == 8) d[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
}

// Zero the border pixels (all c_pad channels) of a spatially padded channels-last copy.
__global__ void __launch_bounds__(256) nhwc_zero_border_kernel(uint4* __restrict__ dst, uint32_t vec_per_px,
                                                               uint32_t hp, uint32_t wp, uint32_t pad,
                                                               uint64_t total_px) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total_px * vec_per_px;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t px = i / vec_per_px;
    const uint32_t x = static_cast<uint32_t>(px % wp), y = static_cast<uint32_t>((px / wp) % hp);
    if (y < pad || y >= hp - pad || x < pad || x >= wp - pad) dst[i] = make_uint4(0, 0, 0, 0);
  }
}

struct FusedArgs {
  float* __restrict__ out;
  uint32_t n_img, h_out, w_out, hw, co;
  uint32_t box_w, box_h, box_n;
  uint32_t ow_tiles, oh_tiles, n_tiles, co_tiles;
  uint32_t k_slabs, fh_slabs;  // k_slabs = Hf * fh_slabs
  uint32_t group;              // consecutive tiles per CTA visit (the pieces of an output row together)
};

// This CTA's tiles: runs of `group` consecutive tiles, runs strided by the grid (group 1 =
// the plain grid stride).  A CTA writing neighbouring pieces of the same NCHW rows back to
// back raises the output write rate (tools/probes/nchw_store_probe.cu: 2.4 -> 3.1-3.5 TB/s).
struct TileWalk {
  uint32_t t, i, group, jump;
  IM2WIN_DEVICE explicit TileWalk(uint32_t g)
      : t(blockIdx.x * g), i(0), group(g), jump((gridDim.x - 1) * g + 1) {}
  IM2WIN_DEVICE void next() {
    if (++i == group) {
      i = 0;
      t += jump;
    } else {
      ++t;
    }
  }
};

// RB: the whole packed filter (k_slabs tiles of N x 128 B) is loaded once per CTA and
// stays resident; only window tiles stream through the ring (small filters: the
// 3-channel input layers, where staging the filter per tile doubles the TMA rows).
//
// ROW = 64: 64-byte K rows (SW64) instead of 128 (SW128), for inputs whose window row Wf * C_pad
// fits in 64 bytes (conv7: 3 taps x 8 bf16 channels = 48 B) -- half the TMA bytes and half the
// MMAs of 128-byte rows, most of which are channel padding there.
template <bool BF16, int N, int STAGES, bool RB = false, int ROW = 128>
__global__ void __launch_bounds__(kTcThreadsFeed, 1)
    conv_tc_fused_kernel(const FusedArgs a, const __grid_constant__ CUtensorMap tmap_a,
                         const __grid_constant__ CUtensorMap tmap_b, const NhwcFeed feed) {
  constexpr uint32_t kRowB = ROW;
  constexpr uint32_t kABytes = kTileM * kRowB;
  constexpr uint32_t kBBytes = RB ? 0 : N * kRowB;
  constexpr uint32_t kStageBytes = kABytes + kBBytes;
  constexpr int kBK = (BF16 ? 64 : 32) * ROW / 128;
  constexpr int kUK = BF16 ? 16 : 8;
  constexpr uint32_t kTmemCols = (2 * N <= 128) ? 128 : (2 * N <= 256 ? 256 : 512);
  constexpr uint32_t kIdesc = instr_desc<BF16, N>();

  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2];
  __shared__ __align__(8) uint64_t tempty_bar[2];
  __shared__ __align__(8) uint64_t bres_bar;
  __shared__ uint32_t tmem_base_sh;

  uint8_t* smem_base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t pix_per_tile = a.box_w * a.box_h * a.box_n;
  const uint32_t a_box_bytes = pix_per_tile * kRowB;
  // RB: resident filter tiles first, then the A ring
  const uint32_t rb_bytes = RB ? a.k_slabs * N * kRowB : 0;
  uint8_t* smem = smem_base + rb_bytes;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&bres_bar, 1);
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
          tma_load_2d(smem_base + ks * N * kRowB, &tmap_b, &bres_bar, ks * kBK, 0);
      }
      uint32_t conf_lo = 1, conf_hi = 0;
      for (TileWalk w(a.group); w.t < total_tiles; w.next()) {
        const uint32_t t = w.t;
        const uint32_t co_blk = t % a.co_tiles;
        uint32_t pt = t / a.co_tiles;
        const uint32_t ow0 = (pt % a.ow_tiles) * a.box_w;
        pt /= a.ow_tiles;
        const uint32_t oh0 = (pt % a.oh_tiles) * a.box_h;
        const uint32_t n0 = (pt / a.oh_tiles) * a.box_n;
        nhwc_feed_wait(feed, n0, n0 + a.box_n - 1, conf_lo, conf_hi);
        for (uint32_t ks = 0; ks < a.k_slabs; ++ks) {
          const uint32_t fh = ks / a.fh_slabs;
          const uint32_t j0 = (ks % a.fh_slabs) * kBK;
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * kStageBytes;
          mbar_arrive_expect_tx(&full_bar[stage], a_box_bytes + kBBytes);
          asm volatile(
              "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, "
              "%7}], [%2];\n" ::"r"(smem_u32(st)),
              "l"(&tmap_a), "r"(smem_u32(&full_bar[stage])), "r"(j0), "r"(fh), "r"(ow0), "r"(oh0), "r"(n0)
              : "memory");
          if constexpr (!RB) tma_load_2d(st + kABytes, &tmap_b, &full_bar[stage], ks * kBK, co_blk * N);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      if constexpr (RB) mbar_wait(&bres_bar, 0);
      for (TileWalk w(a.group); w.t < total_tiles; w.next()) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * N;
        for (uint32_t ks = 0; ks < a.k_slabs; ++ks) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t abase = smem_u32(smem + stage * kStageBytes);
          const uint32_t bbase = RB ? smem_u32(smem_base) + ks * N * kRowB : abase + kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / kUK; ++kk)
            mma<BF16>(tmem_d, smem_desc_row<ROW>(abase + kk * 32), smem_desc_row<ROW>(bbase + kk * 32), kIdesc,
                      (ks | kk) != 0);
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
    const uint32_t r_w = r % a.box_w, r_h = (r / a.box_w) % a.box_h, r_n = r / (a.box_w * a.box_h);
    uint32_t acc = 0, acc_phase = 0;
    for (TileWalk w(a.group); w.t < total_tiles; w.next()) {
      const uint32_t t = w.t;
      const uint32_t co_blk = t % a.co_tiles;
      uint32_t pt = t / a.co_tiles;
      const uint32_t ow = (pt % a.ow_tiles) * a.box_w + r_w;
      pt /= a.ow_tiles;
      const uint32_t oh = (pt % a.oh_tiles) * a.box_h + r_h;
      const uint32_t img = (pt / a.oh_tiles) * a.box_n + r_n;
      const bool valid = r < pix_per_tile && ow < a.w_out && oh < a.h_out && img < a.n_img;
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

// B[m][fh*Kfh + j] = F[m][c][fh][fw] for j = fw*CP + c (c < C real channels, CP = padded
// channel pitch of the NHWC copy), zero elsewhere.
template <bool BF16>
__global__ void pack_filter_fused_kernel(const float* __restrict__ flt, void* __restrict__ packed, int M, int C,
                                         int CP, int h_f, int w_f, int Mp, int Kfh, int Kp) {
  const int64_t total = static_cast<int64_t>(Mp) * Kp;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i / Kp);
    const int kp = static_cast<int>(i % Kp);
    const int fh = kp / Kfh, j = kp % Kfh;
    float v = 0.0f;
    const int fw = j / CP, c = j % CP;
    if (m < M && fw < w_f && c < C) v = flt[((static_cast<int64_t>(m) * C + c) * h_f + fh) * w_f + fw];
    if constexpr (BF16) {
      reinterpret_cast<__nv_bfloat16*>(packed)[i] = __float2bfloat16_rn(v);
    } else {
      uint32_t r;
      asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(v));
      reinterpret_cast<uint32_t*>(packed)[i] = r;
    }
  }
}

template <bool BF16, int N, int STAGES, bool RB = false, int ROW = 128>
static int launch_fused(FusedArgs a, const void* x_cl, const void* packed, int64_t c_in, int64_t h, int64_t w,
                        int32_t h_f, int32_t w_f, int32_t stride, int64_t Kp, int64_t Mp, const NhwcFeed& feed,
                        cudaStream_t stream, const char** err) {
  constexpr int kBK = (BF16 ? 64 : 32) * ROW / 128;
  constexpr CUtensorMapSwizzle kSwz = ROW == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  auto enc = get_encode_fn();
  if (!enc) {
    *err = "conv_tc_fused: cuTensorMapEncodeTiled unavailable";
    return 2;
  }
  const cuuint64_t esz = BF16 ? 2 : 4;
  const CUtensorMapDataType dt = BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUtensorMap map_a, map_b;
  {
    cuuint64_t dims[5] = {static_cast<cuuint64_t>(w_f) * c_in, static_cast<cuuint64_t>(h_f), a.w_out, a.h_out,
                          a.n_img};
    cuuint64_t strides[4] = {static_cast<cuuint64_t>(w) * c_in * esz, static_cast<cuuint64_t>(stride) * c_in * esz,
                             static_cast<cuuint64_t>(stride) * w * c_in * esz,
                             static_cast<cuuint64_t>(h) * w * c_in * esz};
    cuuint32_t box[5] = {static_cast<cuuint32_t>(kBK), 1, a.box_w, a.box_h, a.box_n};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(&map_a, dt, 5, const_cast<void*>(x_cl), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     kSwz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      *err = "conv_tc_fused: window tensor map rejected (cuTensorMapEncodeTiled)";
      return 2;
    }
  }
  {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(Mp)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(Kp) * esz};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(N)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&map_b, dt, 2, const_cast<void*>(packed), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     kSwz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      *err = "conv_tc_fused: filter tensor map rejected (cuTensorMapEncodeTiled)";
      return 2;
    }
  }
  a.co_tiles = static_cast<uint32_t>(Mp / N);
  {
    // runs of consecutive tiles per CTA when an output row is split into several pieces
    const char* g_env = getenv("IM2WIN_TILE_GROUP");
    const uint64_t tiles = static_cast<uint64_t>(a.n_tiles) * a.oh_tiles * a.ow_tiles * a.co_tiles;
    // measured (conv7, 2 pieces per row): runs of 3-4 tiles 28.9 -> 31.4 TF; only with >= 32 runs per CTA
    const int g = g_env ? atoi(g_env) : (a.ow_tiles > 1 && a.co_tiles == 1 && tiles >= 4ull * 32 * 148 ? 4 : 1);
    a.group = static_cast<uint32_t>(g < 1 ? 1 : g);
  }
  const size_t rb = RB ? static_cast<size_t>(a.k_slabs) * N * ROW : 0;
  const size_t smem = rb + static_cast<size_t>(STAGES) * (kTileM + (RB ? 0 : N)) * ROW + 1024;
  auto kern = conv_tc_fused_kernel<BF16, N, STAGES, RB, ROW>;
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
  if (ROW == 64)
    im2win_note_kernel(BF16 ? "conv_tc_fused_kernel (generic TMA window boxes, filter resident, 64-byte rows, bf16)"
                            : "conv_tc_fused_kernel (generic TMA window boxes, filter resident, 64-byte rows, tf32)");
  else
  im2win_note_kernel(RB ? (BF16 ? "conv_tc_fused_kernel (generic TMA window boxes, filter resident, bf16)"
                              : "conv_tc_fused_kernel (generic TMA window boxes, filter resident, tf32)")
                     : (BF16 ? "conv_tc_fused_kernel (generic TMA window boxes, bf16)"
                             : "conv_tc_fused_kernel (generic TMA window boxes, tf32)"));
  e = launch_tc_kernel(kern, grid, smem, stream, feed.src != nullptr, 1, a, map_a, map_b, feed_for(feed, grid, tiles));
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 2;
  }
  return 0;
}

}  // namespace tc
}  // namespace im2win

// Channel pitch of the NHWC copy: the smallest 16-byte multiple >= c (TMA stride rule).
int64_t im2win_nhwc_channel_pitch(int64_t c, int bf16) {
  const int64_t q = bf16 ? 8 : 4;
  return (c + q - 1) / q * q;
}

namespace im2win {
namespace tc {
// The feed warps' code alone (no conv): tools/feed_ab.py measures its copy rate (IM2WIN_FEED_PROBE=1).
template <bool BF16>
__global__ void __launch_bounds__(32 * kFeedWarps) nhwc_feed_only_kernel(const NhwcFeed f) {
  nhwc_feed_run<BF16>(f, threadIdx.x % 32, blockIdx.x * kFeedWarps + threadIdx.x / 32, gridDim.x * kFeedWarps);
}
}  // namespace tc
}  // namespace im2win

int im2win_launch_nchw_to_nhwc(const float* src, void* dst, int64_t n, int64_t c, int64_t h, int64_t w, int bf16,
                               int pad, cudaStream_t stream, const char** err) {
  if (pad == 0 && getenv("IM2WIN_FEED_PROBE") && atoi(getenv("IM2WIN_FEED_PROBE")) > 0) {
    using namespace im2win::tc;
    static uint32_t* counters = nullptr;
    static int64_t cap = 0;
    if (cap < n + 1) {
      if (counters) cudaFree(counters);
      cudaMalloc(&counters, (n + 1) * 4);
      cap = n + 1;
    }
    NhwcFeed feed{};
    feed.src = src;
    feed.dst = dst;
    feed.c_in = static_cast<uint32_t>(c);
    feed.c_pad = static_cast<uint32_t>(im2win_nhwc_channel_pitch(c, bf16));
    feed.hw = static_cast<uint32_t>(h * w);
    feed.n_img = static_cast<uint32_t>(n);
    const uint32_t pix = bf16 ? FeedShape<true>::kPix : FeedShape<false>::kPix;
    const uint32_t grp = bf16 ? FeedShape<true>::G : FeedShape<false>::G;
    feed.chunks = static_cast<uint32_t>((h * w + pix - 1) / pix);
    feed.units_per_img = feed.chunks * ((feed.c_pad + grp - 1) / grp);
    feed.ready = counters;
    feed.front = counters + n;
    feed.lookahead = 0xffffffffu;  // no conv to follow
    cudaMemsetAsync(counters, 0, (n + 1) * 4, stream);
    const int g = atoi(getenv("IM2WIN_FEED_PROBE"));  // CTAs of kFeedWarps warps
    if (bf16) nhwc_feed_only_kernel<true><<<g, 32 * kFeedWarps, 0, stream>>>(feed);
    else nhwc_feed_only_kernel<false><<<g, 32 * kFeedWarps, 0, stream>>>(feed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { *err = cudaGetErrorString(e); return 2; }
    return 0;
  }
  using im2win::tc::PadMap;
  const int64_t hw = h * w;
  const int64_t cp = im2win_nhwc_channel_pitch(c, bf16);
  const int64_t hw_tiles = (hw + 31) / 32, c_tiles = (cp + 31) / 32;
  const int64_t total = n * hw_tiles * c_tiles;
  const int64_t hp = h + 2 * pad, wp = w + 2 * pad;
  if (total >= (1ll << 32) || hw >= (1ll << 31) || hp * wp >= (1ll << 31)) {
    *err = "nchw_to_nhwc: extents exceed the kernel's index range";
    return 1;
  }
  if ((reinterpret_cast<uintptr_t>(dst) & 15) != 0 || (reinterpret_cast<uintptr_t>(src) & 3) != 0) {
    *err = "nchw_to_nhwc: dst must be 16-byte aligned and src 4-byte aligned";
    return 1;
  }
  PadMap pm;
  pm.pad = static_cast<uint32_t>(pad);
  pm.wp = static_cast<uint32_t>(wp);
  pm.img_px = static_cast<uint64_t>(hp * wp);
  pm.fd_w = im2win::FastDiv(static_cast<uint32_t>(w));
  auto done = [&]() -> int {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      *err = cudaGetErrorString(e);
      return 2;
    }
    return 0;
  };
  if (pad > 0) {
    // border pixels: zeros across the whole channel pitch (cp * esz is a 16-byte multiple)
    const uint32_t vec = static_cast<uint32_t>(cp * (bf16 ? 2 : 4) / 16);
    const uint64_t px = static_cast<uint64_t>(n) * hp * wp;
    const uint32_t g = static_cast<uint32_t>(std::min<uint64_t>((px * vec + 255) / 256, 148 * 16));
    im2win::tc::nhwc_zero_border_kernel<<<g, 256, 0, stream>>>(static_cast<uint4*>(dst), vec,
                                                               static_cast<uint32_t>(hp), static_cast<uint32_t>(wp),
                                                               static_cast<uint32_t>(pad), px);
  }
  if (cp <= 8) {
    const uint64_t pixels = static_cast<uint64_t>(n) * hw;
    const uint32_t g = static_cast<uint32_t>(std::min<uint64_t>((pixels + 255) / 256, 148 * 32));
    if (bf16)
      im2win::tc::nchw_to_nhwc_small_kernel<true><<<g, 256, 0, stream>>>(src, dst, static_cast<uint32_t>(c),
                                                                         static_cast<uint32_t>(cp), hw, pixels, pm);
    else
      im2win::tc::nchw_to_nhwc_small_kernel<false><<<g, 256, 0, stream>>>(src, dst, static_cast<uint32_t>(c),
                                                                          static_cast<uint32_t>(cp), hw, pixels, pm);
    return done();
  }
  if (hw % 4 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    const int64_t wt = n * ((hw + 63) / 64) * ((cp + 63) / 64);
    if (wt < (1ll << 32)) {
      const uint32_t g = static_cast<uint32_t>(std::min<int64_t>(wt, 148 * 8));
      if (bf16)
        im2win::tc::nchw_to_nhwc_wide_kernel<true><<<g, 256, 0, stream>>>(
            src, dst, static_cast<uint32_t>(c), static_cast<uint32_t>(cp), static_cast<uint32_t>(hw),
            static_cast<uint32_t>((hw + 63) / 64), static_cast<uint32_t>((cp + 63) / 64), static_cast<uint32_t>(wt), pm);
      else
        im2win::tc::nchw_to_nhwc_wide_kernel<false><<<g, 256, 0, stream>>>(
            src, dst, static_cast<uint32_t>(c), static_cast<uint32_t>(cp), static_cast<uint32_t>(hw),
            static_cast<uint32_t>((hw + 63) / 64), static_cast<uint32_t>((cp + 63) / 64), static_cast<uint32_t>(wt), pm);
      return done();
    }
  }
  const char* cbe = getenv("IM2WIN_COPY_BLOCK");  // 0: the 32x32 generic kernel (A/B)
  if (hw <= 256 && !(cbe && atoi(cbe) == 0)) {
    const int64_t bt = n * ((c + 31) / 32);
    if (bt < (1ll << 32)) {
      const uint32_t g = static_cast<uint32_t>(std::min<int64_t>(bt, 148 * 16));
      const uint32_t vec = ((c * hw) % 4 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) ? 1u : 0u;
      const size_t sm = static_cast<size_t>(32) * (hw | 1) * 4;
      if (bf16)
        im2win::tc::nchw_to_nhwc_block_kernel<true><<<g, 128, sm, stream>>>(
            src, dst, static_cast<uint32_t>(c), static_cast<uint32_t>(cp), static_cast<uint32_t>(hw),
            static_cast<uint32_t>((c + 31) / 32), static_cast<uint32_t>(bt), vec, pm);
      else
        im2win::tc::nchw_to_nhwc_block_kernel<false><<<g, 128, sm, stream>>>(
            src, dst, static_cast<uint32_t>(c), static_cast<uint32_t>(cp), static_cast<uint32_t>(hw),
            static_cast<uint32_t>((c + 31) / 32), static_cast<uint32_t>(bt), vec, pm);
      return done();
    }
  }
  const uint32_t grid = static_cast<uint32_t>(total < 148 * 16 ? total : 148 * 16);
  if (bf16)
    im2win::tc::nchw_to_nhwc_kernel<true><<<grid, 256, 0, stream>>>(
        src, dst, static_cast<uint32_t>(c), static_cast<uint32_t>(cp), static_cast<uint32_t>(hw),
        static_cast<uint32_t>(hw_tiles), static_cast<uint32_t>(c_tiles), static_cast<uint32_t>(total), pm);
  else
    im2win::tc::nchw_to_nhwc_kernel<false><<<grid, 256, 0, stream>>>(
        src, dst, static_cast<uint32_t>(c), static_cast<uint32_t>(cp), static_cast<uint32_t>(hw),
        static_cast<uint32_t>(hw_tiles), static_cast<uint32_t>(c_tiles), static_cast<uint32_t>(total), pm);
  return done();
}

size_t im2win_tc_fused_workspace_bytes(int64_t c_in, int64_t c_out, int h_f, int w_f) {
  c_in = im2win_nhwc_channel_pitch(c_in, 1);  // >= either pitch
  const int64_t Mp = (c_out + 255) / 256 * 256 + 256;
  const int64_t Kfh = (w_f * c_in + 63) / 64 * 64;
  const int64_t Kshift = static_cast<int64_t>(w_f) * ((c_in + 63) / 64 * 64);  // window-shift packing
  return static_cast<size_t>(Mp * std::max(Kfh, Kshift) * h_f) * 4 + 1024;
}

// The in-kernel feed's counters (n ready counters + 1 claim counter) follow the packed filter.
uint32_t* im2win_tc_feed_counters(void* workspace, int64_t c_in, int64_t c_out, int h_f, int w_f) {
  return reinterpret_cast<uint32_t*>(static_cast<char*>(workspace) +
                                     im2win_tc_fused_workspace_bytes(c_in, c_out, h_f, w_f));
}

size_t im2win_tc_fused_feed_workspace_bytes(int64_t n, int64_t c_in, int64_t c_out, int h_f, int w_f) {
  return im2win_tc_fused_workspace_bytes(c_in, c_out, h_f, w_f) + static_cast<size_t>(n + 1) * 4 + 256;
}

int im2win_try_conv_tc_shift(const void* x_cl, const float* flt, float* out, void* workspace, int64_t n, int64_t c_in,
                             int64_t c_pad, int64_t h, int64_t w, int64_t c_out, int h_f, int w_f, int stride, int bf16,
                             double fused_util, const im2win::tc::NhwcFeed& feed, cudaStream_t stream,
                             const char** err);

int im2win_try_conv_tc_phase(const void* x_cl, const float* flt, float* out, void* workspace, int64_t n, int64_t c_in,
                             int64_t c_pad, int64_t h, int64_t w, int64_t c_out, int h_f, int w_f, int stride, int bf16,
                             double fused_util, const im2win::tc::NhwcFeed& feed, cudaStream_t stream,
                             const char** err);

int im2win_launch_conv_tc_fused(const void* x_cl, const float* flt, float* out, void* workspace, int64_t n,
                                int64_t c_in, int64_t h, int64_t w, int64_t c_out, int h_f, int w_f, int stride,
                                int bf16, const float* feed_src, cudaStream_t stream, const char** err) {
  using namespace im2win::tc;
  // feed_src != nullptr: x_cl is scratch, produced from the NCHW input inside the conv kernel
  // (counters at the end of the workspace, see im2win_tc_feed_counters)
  NhwcFeed feed{};
  if (feed_src) {
    // In-kernel feed or a copy kernel first.  Measured (tools/feed_ab.py): the feed warps share the
    // SM's L1/shared-memory datapath and HBM with the conv, so overlap pays only where the conv's
    // own traffic is light next to the input -- output/input elements r = (Co*Ho*Wo)/(C*H*W) <= 0.5
    // (strided layers: conv4 N=128 BF16 1.15 -> 1.02 ms, TF32 1.98 -> 1.82 ms) -- and only at small
    // batches (conv4 N=512: BF16 4.48 -> 4.20 but TF32 7.81 -> 7.90; N=2048 slower for both); at
    // r ~ 0.9 (conv9/10) it ties or loses, at r >= 1.4 (conv5/6/8) it loses up to 18%.
    // IM2WIN_FEED: 0 never, 1 auto (r <= 0.5 and N <= 256), 2 always.
    const char* fe = getenv("IM2WIN_FEED");
    const int mode = fe ? atoi(fe) : 1;
    const int64_t h_o = (h - h_f) / stride + 1, w_o = (w - w_f) / stride + 1;
    const double r = static_cast<double>(c_out * h_o * w_o) / static_cast<double>(c_in * h * w);
    if (mode == 0 || (mode == 1 && (r > 0.5 || n > 256))) {
      const int rc = im2win_launch_nchw_to_nhwc(feed_src, const_cast<void*>(x_cl), n, c_in, h, w, bf16, 0, stream, err);
      if (rc) return rc;
      feed_src = nullptr;
    }
  }
  if (feed_src) {
    const int64_t hw = h * w;
    if (hw >= (1ll << 31) || n * ((hw + 63) / 64) * ((c_in + 7) / 8) >= (1ll << 32)) {
      *err = "conv_tc_fused: extents exceed the feed's index range";
      return 1;
    }
    feed.src = feed_src;
    feed.dst = const_cast<void*>(x_cl);
    feed.c_in = static_cast<uint32_t>(c_in);
    feed.c_pad = static_cast<uint32_t>(im2win_nhwc_channel_pitch(c_in, bf16));
    feed.hw = static_cast<uint32_t>(hw);
    feed.n_img = static_cast<uint32_t>(n);
    const uint32_t pix = bf16 ? FeedShape<true>::kPix : FeedShape<false>::kPix;
    const uint32_t grp = bf16 ? FeedShape<true>::G : FeedShape<false>::G;
    feed.chunks = static_cast<uint32_t>((hw + pix - 1) / pix);
    feed.units_per_img = feed.chunks * ((feed.c_pad + grp - 1) / grp);
    feed.ready = im2win_tc_feed_counters(workspace, c_in, c_out, h_f, w_f);
    feed.front = feed.ready + n;
    feed.lookahead = 2;  // set per kernel by the launcher (feed_lookahead)
    feed.nowait = getenv("IM2WIN_FEED_NOWAIT") && atoi(getenv("IM2WIN_FEED_NOWAIT")) ? 1u : 0u;
    cudaError_t e = cudaMemsetAsync(feed.ready, 0, static_cast<size_t>(n + 1) * 4, stream);
    if (e != cudaSuccess) {
      *err = cudaGetErrorString(e);
      return 2;
    }
  }
  const int64_t cp = im2win_nhwc_channel_pitch(c_in, bf16);  // channel pitch of x_cl
  const int64_t h_out = (h - h_f) / stride + 1, w_out = (w - w_f) / stride + 1;
  int N = c_out <= 64 ? 64 : c_out <= 96 ? 96 : c_out <= 128 ? 128 : 256;
  const int bk = bf16 ? 64 : 32;
  const int64_t Kfh = (w_f * cp + bk - 1) / bk * bk;
  const int64_t Kp = Kfh * h_f;
  FusedArgs a{};
  a.out = out;
  a.n_img = static_cast<uint32_t>(n);
  a.h_out = static_cast<uint32_t>(h_out);
  a.w_out = static_cast<uint32_t>(w_out);
  a.hw = static_cast<uint32_t>(h_out * w_out);
  a.co = static_cast<uint32_t>(c_out);
  if (w_out > kTileM) {
    const int64_t parts = (w_out + kTileM - 1) / kTileM;
    a.box_w = static_cast<uint32_t>((w_out + parts - 1) / parts);
    a.box_h = 1;
    a.box_n = 1;
  } else {
    a.box_w = static_cast<uint32_t>(w_out);
    a.box_h = static_cast<uint32_t>(std::min<int64_t>(h_out, kTileM / w_out));
    a.box_n = a.box_h == h_out ? static_cast<uint32_t>(std::min<int64_t>(n, kTileM / (w_out * h_out))) : 1u;
  }
  a.ow_tiles = (a.w_out + a.box_w - 1) / a.box_w;
  a.oh_tiles = (a.h_out + a.box_h - 1) / a.box_h;
  a.n_tiles = (a.n_img + a.box_n - 1) / a.box_n;
  {
    // few pixel tiles (conv12 at N=128: 26 tiles of 125 pixels): narrower Co tiles put more
    // CTAs on the SMs (each re-reads its A tiles from L2)
    static thread_local int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (sms <= 0) sms = 148;
    }
    const char* ne = getenv("IM2WIN_FUSED_NARROW");
    const uint64_t ptiles = static_cast<uint64_t>(a.ow_tiles) * a.oh_tiles * a.n_tiles;
    // (not below 128: a 128x64 UMMA is shared-memory bound -- conv12 at N = 64 measured 224 vs 274 TF)
    if (!(ne && atoi(ne) == 0) && N == 256 &&
        ptiles * static_cast<uint64_t>((c_out + N - 1) / N) < static_cast<uint64_t>(sms))
      N = 128;
  }
  const int64_t Mp = (c_out + N - 1) / N * N;
  a.fh_slabs = static_cast<uint32_t>(Kfh / bk);
  a.k_slabs = a.fh_slabs * h_f;
  // 64-byte K rows when a filter row's window (Wf * C_pad elements) fits in 64 bytes and the filter
  // stays resident (conv7: BF16 0.656 -> 0.596 ms at N=128, same bits -- the box rows, not their
  // bytes, bound this layer); IM2WIN_ROW64=0 keeps 128-byte rows
  const int64_t esz = bf16 ? 2 : 4;
  const char* r64e = getenv("IM2WIN_ROW64");
  const bool row64 = !(r64e && atoi(r64e) == 0) && w_f * cp * esz <= 64 && Mp == N && N <= 128;
  const int bk64 = bf16 ? 32 : 16;
  {
    // the phase kernel reuses each loaded A tile for every tap of a stride phase (any stride <= 2)
    const double util = static_cast<double>(a.box_w) * a.box_h * a.box_n / kTileM;
    const int rc = im2win_try_conv_tc_phase(x_cl, flt, out, workspace, n, c_in, cp, h, w, c_out, h_f, w_f, stride,
                                            bf16, util, feed, stream, err);
    if (rc != 0) return rc > 0 ? 0 : -rc;
  }
  {
    // stride-1 layers: the window-shift kernel reuses each loaded A tile for all Wf taps
    const double util = static_cast<double>(a.box_w) * a.box_h * a.box_n / kTileM;
    const int rc = im2win_try_conv_tc_shift(x_cl, flt, out, workspace, n, c_in, cp, h, w, c_out, h_f, w_f, stride,
                                            bf16, util, feed, stream, err);
    if (rc != 0) return rc > 0 ? 0 : -rc;
  }
  if (row64) {
    // one 64-byte slab per filter row: repack with Kfh = 32 (bf16) / 16 (tf32) and launch
    FusedArgs b = a;
    b.fh_slabs = 1;
    b.k_slabs = static_cast<uint32_t>(h_f);
    const int64_t Kp64 = static_cast<int64_t>(bk64) * h_f;
    if (bf16)
      pack_filter_fused_kernel<true><<<256, 256, 0, stream>>>(flt, workspace, static_cast<int>(c_out),
                                                              static_cast<int>(c_in), static_cast<int>(cp), h_f, w_f,
                                                              static_cast<int>(Mp), bk64, static_cast<int>(Kp64));
    else
      pack_filter_fused_kernel<false><<<256, 256, 0, stream>>>(flt, workspace, static_cast<int>(c_out),
                                                               static_cast<int>(c_in), static_cast<int>(cp), h_f, w_f,
                                                               static_cast<int>(Mp), bk64, static_cast<int>(Kp64));
#define IM2WIN_FU64(BF, NN) \
  return launch_fused<BF, NN, 8, true, 64>(b, x_cl, workspace, cp, h, w, h_f, w_f, stride, Kp64, Mp, feed, stream, err)
    if (bf16) {
      if (N == 64) IM2WIN_FU64(true, 64);
      if (N == 96) IM2WIN_FU64(true, 96);
      IM2WIN_FU64(true, 128);
    } else {
      if (N == 64) IM2WIN_FU64(false, 64);
      if (N == 96) IM2WIN_FU64(false, 96);
      IM2WIN_FU64(false, 128);
    }
#undef IM2WIN_FU64
  }
  if (bf16)
    pack_filter_fused_kernel<true><<<256, 256, 0, stream>>>(flt, workspace, static_cast<int>(c_out),
                                                            static_cast<int>(c_in), static_cast<int>(cp), h_f, w_f,
                                                            static_cast<int>(Mp), static_cast<int>(Kfh),
                                                            static_cast<int>(Kp));
  else
    pack_filter_fused_kernel<false><<<256, 256, 0, stream>>>(flt, workspace, static_cast<int>(c_out),
                                                             static_cast<int>(c_in), static_cast<int>(cp), h_f, w_f,
                                                             static_cast<int>(Mp), static_cast<int>(Kfh),
                                                             static_cast<int>(Kp));
#define IM2WIN_FU(BF, NN, ST) \
  return launch_fused<BF, NN, ST>(a, x_cl, workspace, cp, h, w, h_f, w_f, stride, Kp, Mp, feed, stream, err)
#define IM2WIN_FU_RB(BF, NN) \
  return launch_fused<BF, NN, 6, true>(a, x_cl, workspace, cp, h, w, h_f, w_f, stride, Kp, Mp, feed, stream, err)
  {
    // filter-resident mode: one Co tile whose whole packed filter fits beside 6 window stages
    const char* rb_env = getenv("IM2WIN_FUSED_RB");
    const size_t rb_bytes = static_cast<size_t>(a.k_slabs) * N * kRowBytes;
    const bool rb = Mp == N && (N == 64 || N == 96 || N == 128) &&
                    rb_bytes + 6 * kTileM * kRowBytes + 1024 <= 227 * 1024 && !(rb_env && atoi(rb_env) == 0);
    if (rb) {
      if (bf16) {
        switch (N) {
          case 64: IM2WIN_FU_RB(true, 64);
          case 96: IM2WIN_FU_RB(true, 96);
          default: IM2WIN_FU_RB(true, 128);
        }
      } else {
        switch (N) {
          case 64: IM2WIN_FU_RB(false, 64);
          case 96: IM2WIN_FU_RB(false, 96);
          default: IM2WIN_FU_RB(false, 128);
        }
      }
    }
  }
#undef IM2WIN_FU_RB
  if (bf16) {
    switch (N) {
      case 64: IM2WIN_FU(true, 64, 8);
      case 96: IM2WIN_FU(true, 96, 6);
      case 128: IM2WIN_FU(true, 128, 6);
      default: IM2WIN_FU(true, 256, 4);
    }
  } else {
    switch (N) {
      case 64: IM2WIN_FU(false, 64, 8);
      case 96: IM2WIN_FU(false, 96, 6);
      case 128: IM2WIN_FU(false, 128, 6);
      default: IM2WIN_FU(false, 256, 4);
    }
  }
#undef IM2WIN_FU
}
