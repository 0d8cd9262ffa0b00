// Direct tensor-core convolution for few-channel inputs (the RGB layers conv1-3, conv7):
// the im2win transform happens inside the SM.
//
// For C <= 16 the channels-last / TMA-box route moves 128-byte rows that are mostly
// padding (a window row of a 3-channel input is 3*Wf values), and the TMA engine's
// row rate, not the tensor core, bounds the kernel.  Here producer warps stage the
// input patch a tile needs (C x rows x cols, straight from NCHW, coalesced) in
// shared memory and write each output pixel's whole window -- K = C*Hf*Wf values
// in the reference's k order (c, fh, fw), i.e. the im2win window of that pixel
// (layouts.py:73-83) -- as one row of the 128-byte-swizzled K-major A operand.
// The packed filter stays resident in shared memory; a single thread issues
// tcgen05.mma into double-buffered TMEM accumulators; 8 epilogue warps store NCHW.
//
// Warps 0-7: producers (two threads per A row = output pixel, four 16-byte chunks each);
// warp 8: MMA issuer; warp 9: TMEM allocator; warps 12-15: epilogue (one per TMEM lane quarter).
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "tc_common.cuh"

namespace im2win {
namespace tc {

#ifndef IM2WIN_DIRECT_PROD_WARPS
#define IM2WIN_DIRECT_PROD_WARPS 8
#endif
// warps [0, P): producers; P: MMA issuer; P+1: TMEM allocator (+ loader); P+1..P+3: patch
// loaders (BF16); the last 4: epilogue (warp % 4 = TMEM lane quarter).
constexpr int kProdWarps = IM2WIN_DIRECT_PROD_WARPS;
constexpr int kProducers = kProdWarps * 32;
constexpr int kDirWarps = kProdWarps + 8;
constexpr int kDirThreads = kDirWarps * 32;
constexpr int kChunksPerThread = 8 * kTileM / kProducers;  // 16-byte chunks of its A row per slab
static_assert(kDirWarps % 4 == 0, "the epilogue warps must cover the four TMEM lane quarters");
constexpr int kDirEpiWarps = 4;
constexpr int kDirColIters = 16;  // patch rows up to 512 floats (checked by plan_direct)
#ifndef IM2WIN_DIRECT_LOADERS
#define IM2WIN_DIRECT_LOADERS 1  // BF16: warps 9-11 fetch the input patches (mbarrier ring), producers only build
#endif
constexpr int kLoadWarps = 3;
#ifndef IM2WIN_DIRECT_SPLIT_BUILD
#define IM2WIN_DIRECT_SPLIT_BUILD 1  // padded-k check only in the last slab
#endif

struct DirectArgs {
  const float* __restrict__ x;   // NCHW input
  const void* __restrict__ bpk;  // packed filter [Np][Kp] (bf16 or tf32 bits), Kp = slabs * BK
  float* __restrict__ out;       // NCHW output
  uint32_t n_img, c_in, h_in, w_in, h_out, w_out, hw, co, stride, h_f, w_f;
  uint32_t box_w, rows;          // tile = rows x box_w output pixels (<= 128)
  uint32_t ow_tiles, oh_tiles, tiles;
  uint32_t K, slabs, kp;         // K = C*Hf*Wf; kp = slabs * BK (packed row length)
  uint32_t prow, pcol;           // staged patch: prow input rows x pcol input columns per channel
  uint32_t patch_bufs;           // 1 or 2 patch buffers
  uint32_t pad;                  // zero padding on every side
  uint32_t pcolq, prow_pitch;    // patch columns per stride phase; floats per patch row (= stride * pcolq)
};

IM2WIN_DEVICE void named_sync_producers() { asm volatile("bar.sync 1, %0;\n" ::"n"(kProducers) : "memory"); }
IM2WIN_DEVICE void sts32(uint32_t addr, float v) { asm volatile("st.shared.f32 [%0], %1;\n" ::"r"(addr), "f"(v) : "memory"); }
IM2WIN_DEVICE void sts32i(uint32_t addr, int v) { asm volatile("st.shared.b32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory"); }
IM2WIN_DEVICE void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
// Volatile (kept in program order after the barriers) but without a memory clobber, so the
// loads of one chunk are issued back to back and overlap in the LSU.
IM2WIN_DEVICE float lds32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v) : "r"(addr));
  return v;
}
IM2WIN_DEVICE int4 lds128i(uint32_t addr) {
  int4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// Patch columns are read in natural order (lane = column: coalesced) and stored phase-major
// (column s*q + ph at ph*pcolq + q) so lanes later read consecutive words.  The smem offset
// of column lane + 32*i is the same for every row of every tile: computed once per thread.
struct PatchLanes {
  uint32_t dst[kDirColIters];
  uint32_t live;  // bit i: column lane + 32*i lies inside the patch row
  IM2WIN_DEVICE PatchLanes(const DirectArgs& a, uint32_t lane) : live(0) {
#pragma unroll
    for (int i = 0; i < kDirColIters; ++i) {
      const uint32_t col = lane + 32 * i;
      dst[i] = 4 * ((col % a.stride) * a.pcolq + col / a.stride);
      if (col < a.prow_pitch) live |= 1u << i;
    }
  }
};

// Rows w0, w0 + nw, ... of tile t's input patch -> shared buffer `pb` (4-byte cp.async,
// zero-filled outside the image).
IM2WIN_DEVICE void issue_patch_rows(const DirectArgs& a, const PatchLanes& pl, uint32_t t, uint32_t pb, uint32_t w0,
                                    uint32_t nw, uint32_t lane) {
  const uint32_t owt = t % a.ow_tiles;
  const uint32_t rest = t / a.ow_tiles;
  const uint32_t oh0 = (rest % a.oh_tiles) * a.rows;
  const uint32_t img = rest / a.oh_tiles;
  const int ih0 = static_cast<int>(oh0 * a.stride) - static_cast<int>(a.pad);
  const int iw0 = static_cast<int>(owt * a.box_w * a.stride) - static_cast<int>(a.pad);
  const float* xi = a.x + static_cast<int64_t>(img) * a.c_in * a.h_in * a.w_in;
  uint32_t col_in = 0;  // bit i: column lane + 32*i is inside the image (this tile)
#pragma unroll
  for (int i = 0; i < kDirColIters; ++i) {
    const int iw = iw0 + static_cast<int>(lane + 32 * i);
    if (iw >= 0 && iw < static_cast<int>(a.w_in)) col_in |= 1u << i;
  }
  col_in &= pl.live;
  const uint32_t prows_total = a.c_in * a.prow;
  uint32_t c = w0 / a.prow, rr = w0 % a.prow;
  for (uint32_t pr = w0; pr < prows_total; pr += nw) {
    const int ih = ih0 + static_cast<int>(rr);
    const bool in_row = ih >= 0 && ih < static_cast<int>(a.h_in);
    const uint32_t m = in_row ? col_in : 0u;
    const float* src = xi + (static_cast<int64_t>(c) * a.h_in + (in_row ? ih : 0)) * a.w_in + iw0 + lane;
    const uint32_t dst_row = pb + pr * a.prow_pitch * 4;
#pragma unroll
    for (int i = 0; i < kDirColIters; ++i) {
      if ((pl.live >> i) & 1u) {
        const bool ok = (m >> i) & 1u;
        cp_async_4_zfill(dst_row + pl.dst[i], ok ? src + 32 * i : xi, !ok);
      }
    }
    rr += nw;
    while (rr >= a.prow) {
      rr -= a.prow;
      ++c;
    }
  }
}

template <bool BF16, int N, int STAGES>
__global__ void __launch_bounds__(kDirThreads, 1) conv_tc_direct_kernel(const DirectArgs a) {
  constexpr int kBK = BF16 ? 64 : 32;
  constexpr int kUK = BF16 ? 16 : 8;
  constexpr int kPerChunk = BF16 ? 8 : 4;  // elements per 16-byte chunk
  constexpr uint32_t kATile = kTileM * kRowBytes;
  constexpr uint32_t kTmemCols = (2 * N <= 128) ? 128 : (2 * N <= 256 ? 256 : 512);
  constexpr uint32_t kIdesc = instr_desc<BF16, N>();
  // measured (tools/direct_ab.py, N=128): loader warps +7% (conv1) to +22% (conv7) for BF16;
  // TF32 (twice the slabs: the build is the bound) loses 11%, so it keeps in-line fetching
  constexpr bool kLoaders = IM2WIN_DIRECT_LOADERS && BF16;

  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t a_full[STAGES];
  __shared__ __align__(8) uint64_t a_empty[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2];
  __shared__ __align__(8) uint64_t tempty_bar[2];
  __shared__ __align__(8) uint64_t b_ready;
  __shared__ __align__(8) uint64_t p_full[4];   // patch buffer landed (loader threads' cp.async)
  __shared__ __align__(8) uint64_t p_empty[4];  // patch buffer built from (producer warps)
  __shared__ uint32_t tmem_base_sh;

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a_ring = smem;                                        // STAGES x 16 KB
  uint8_t* b_res = a_ring + STAGES * kATile;                     // slabs x N x 128 B
  // per-k patch offsets (kp ints), then the patch buffers (bufs x C x prow x prow_pitch floats)
  const uint32_t koff_s = smem_u32(b_res + a.slabs * N * kRowBytes);
  const uint32_t patch_s = koff_s + ((a.kp * 4 + 15) & ~15u);
  const uint32_t patch_elems = a.c_in * a.prow * a.prow_pitch;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&a_full[s], kProdWarps);
      mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], kDirEpiWarps);
    }
    mbar_init(&b_ready, kProdWarps);
    for (int b = 0; b < 4; ++b) {
      mbar_init(&p_full[b], kLoadWarps * 32);
      mbar_init(&p_empty[b], kProdWarps);
    }
    fence_barrier_init();
  }
  if (warp == kProdWarps + 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_sh)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  if (warp < kProdWarps) {
    // ------------------------------------------------------------- producers
    const uint32_t tid = threadIdx.x;
    const uint32_t arow_i = tid % kTileM, half = tid / kTileM;  // A row, chunk group (j = kCPT*half + jj)
    // resident filter: slab sl, row m, 16-byte chunk j -> swizzled chunk j ^ (m & 7)
    {
      const uint4* src = static_cast<const uint4*>(a.bpk);
      const uint32_t chunks_per_row = a.kp / kPerChunk;
      const uint32_t b_s = smem_u32(b_res);
      for (uint32_t i = tid; i < N * chunks_per_row; i += kProducers) {
        const uint32_t m = i / chunks_per_row, cj = i % chunks_per_row;
        const uint32_t sl = cj / 8, j = cj % 8;
        sts128(b_s + (sl * N + m) * kRowBytes + ((j ^ (m & 7)) << 4), __ldg(src + i));
      }
      // window offsets: k = (c, fh, fw) -> patch[c][fh][phase fw%s][fw/s] relative to the pixel's base
      for (uint32_t k = tid; k < a.kp; k += kProducers) {
        int o = -1;
        if (k < a.K) {
          const uint32_t c = k / (a.h_f * a.w_f), rem = k % (a.h_f * a.w_f);
          const uint32_t fh = rem / a.w_f, fw = rem % a.w_f;
          o = static_cast<int>((c * a.prow + fh) * a.prow_pitch + (fw % a.stride) * a.pcolq + fw / a.stride);
        }
        sts32i(koff_s + 4 * k, o);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&b_ready);
    }
    named_sync_producers();  // koff table complete
    const uint32_t r_row = arow_i / a.box_w, r_col = arow_i % a.box_w;  // this thread's pixel inside the tile
    const bool row_ok = arow_i < a.rows * a.box_w;
    // pixel (r_row, r_col) reads patch rows r_row*s + fh, columns r_col*s + fw = phase fw%s, index r_col + fw/s
    // rows past the tile's pixels build from pixel 0 (in-bounds reads; the epilogue drops them)
    const uint32_t pix_base = row_ok ? (r_row * a.stride) * a.prow_pitch + r_col : 0u;
    const PatchLanes pl(a, lane);
    auto issue_patch = [&](uint32_t t, uint32_t pb) {
      issue_patch_rows(a, pl, t, pb, warp, kProdWarps, lane);
      cp_async_commit();
    };
    // patch_bufs buffers: the patch of tile it + (bufs - 1) is fetched while tile it is built
    const uint32_t nb = a.patch_bufs;
    auto pbuf = [&](uint32_t i) { return patch_s + (i % nb) * patch_elems * 4; };
    if (!kLoaders)
    for (uint32_t d = 0; d + 1 < nb; ++d) {
      const uint32_t tt = blockIdx.x + d * gridDim.x;
      if (tt < a.tiles) issue_patch(tt, pbuf(d));
      else cp_async_commit();
    }
    if (!kLoaders && nb == 1 && blockIdx.x < a.tiles) issue_patch(blockIdx.x, pbuf(0));
    uint32_t stage = 0, phase = 0, it = 0;
    for (uint32_t t = blockIdx.x; t < a.tiles; t += gridDim.x, ++it) {
      const uint32_t pb = pbuf(it);
      if constexpr (kLoaders) {
        mbar_wait(&p_full[it % nb], (it / nb) & 1);  // this tile's patch has landed
      } else {
      // this tile's group is the oldest pending one: allow nb - 2 newer groups in flight
      if (nb >= 4) cp_async_wait<2>();
      else if (nb == 3) cp_async_wait<1>();
      else cp_async_wait<0>();
      named_sync_producers();  // this tile's patch has landed for every producer
      if (nb > 1) {
        const uint32_t ahead = t + (nb - 1) * gridDim.x;  // buffer (it - 1) % nb: its rows were built
        if (ahead < a.tiles) issue_patch(ahead, pbuf(it + nb - 1));
        else cp_async_commit();
      }
      }
      const uint32_t my_base = pb + 4 * pix_base;
      // one slab: this thread's four 16-byte chunks of its A row; only the last slab holds
      // padded k (offset -1 -> zero), so the others skip the check
      auto build_slab = [&](uint32_t sl, auto check) {
        const uint32_t arow = smem_u32(a_ring + stage * kATile) + arow_i * kRowBytes;
        const uint32_t ko = koff_s + 4 * sl * kBK;
        // chunks in groups of CG: per group three latency levels (the loads are volatile asm,
        // issued in program order) -- every chunk's window offsets (warp-uniform: broadcast
        // loads), then every gather, then the packs and stores.  Measured (tools/direct_ab.py,
        // N=128): TF32 all 4 chunks at once +6-10% over chunk by chunk; BF16 (8 values per
        // chunk) 4 at once -4%, 2 at once -3%, so it stays chunk by chunk.
        constexpr int CG = BF16 ? 1 : kChunksPerThread;
#pragma unroll
        for (int jg = 0; jg < kChunksPerThread; jg += CG) {
          int off[CG][8];
#pragma unroll
          for (int jj = 0; jj < CG; ++jj) {
            const int j = kChunksPerThread * half + jg + jj;
            const int4 o_lo = lds128i(ko + 4 * (j * kPerChunk));
            off[jj][0] = o_lo.x; off[jj][1] = o_lo.y; off[jj][2] = o_lo.z; off[jj][3] = o_lo.w;
            if constexpr (BF16) {
              const int4 o_hi = lds128i(ko + 4 * (j * kPerChunk + 4));
              off[jj][4] = o_hi.x; off[jj][5] = o_hi.y; off[jj][6] = o_hi.z; off[jj][7] = o_hi.w;
            }
          }
          float v[CG][kPerChunk];
#pragma unroll
          for (int jj = 0; jj < CG; ++jj)
#pragma unroll
            for (int e = 0; e < kPerChunk; ++e) {
              if constexpr (decltype(check)::value) v[jj][e] = off[jj][e] >= 0 ? lds32(my_base + 4 * off[jj][e]) : 0.0f;
              else v[jj][e] = lds32(my_base + 4 * off[jj][e]);
            }
#pragma unroll
          for (int jj = 0; jj < CG; ++jj) {
            const int j = kChunksPerThread * half + jg + jj;
            uint32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              w[q] = BF16 ? pack_bf16x2(v[jj][2 * q], v[jj][(2 * q + 1) % kPerChunk]) : to_tf32(v[jj][q]);
            sts128(arow + ((j ^ (arow_i & 7)) << 4), make_uint4(w[0], w[1], w[2], w[3]));
          }
        }
      };
      for (uint32_t sl = 0; sl < a.slabs; ++sl) {
        mbar_wait(&a_empty[stage], phase ^ 1);
#if IM2WIN_DIRECT_SPLIT_BUILD
        if (sl + 1 < a.slabs) build_slab(sl, std::false_type{});
        else build_slab(sl, std::true_type{});
#else
        build_slab(sl, std::true_type{});
#endif
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if constexpr (kLoaders) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_empty[it % nb]);  // this warp's rows are built: buffer reusable
      } else if (nb == 1 && t + gridDim.x < a.tiles) {
        named_sync_producers();  // every row built from the single buffer
        issue_patch(t + gridDim.x, pbuf(0));
      }
    }
  } else if (kLoaders && warp >= kProdWarps + 1 && warp < kProdWarps + 1 + kLoadWarps) {
    // ------------------------------------------------------------- patch loaders
    const PatchLanes pl(a, lane);
    const uint32_t nb = a.patch_bufs;
    uint32_t it = 0;
    for (uint32_t t = blockIdx.x; t < a.tiles; t += gridDim.x, ++it) {
      const uint32_t b = it % nb;
      if (it >= nb) mbar_wait(&p_empty[b], ((it / nb) - 1) & 1);
      issue_patch_rows(a, pl, t, patch_s + b * patch_elems * 4, warp - kProdWarps - 1, kLoadWarps, lane);
      cp_async_arrive_noinc(&p_full[b]);
    }
    cp_async_wait<0>();
  } else if (warp == kProdWarps) {
    // ------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      mbar_wait(&b_ready, 0);
      tc_fence_after();
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      const uint32_t bbase0 = smem_u32(b_res);
      for (uint32_t t = blockIdx.x; t < a.tiles; t += gridDim.x) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * N;
        for (uint32_t sl = 0; sl < a.slabs; ++sl) {
          mbar_wait(&a_full[stage], phase);
          tc_fence_after();
          const uint32_t abase = smem_u32(a_ring + stage * kATile);
          const uint32_t bbase = bbase0 + sl * N * kRowBytes;
#pragma unroll
          for (int kk = 0; kk < kBK / kUK; ++kk)
            mma<BF16>(tmem_d, smem_desc_sw128(abase + kk * 32), smem_desc_sw128(bbase + kk * 32), kIdesc,
                      (sl | kk) != 0);
          mma_commit(&a_empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull_bar[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= kDirWarps - kDirEpiWarps) {
    // ------------------------------------------------------------- epilogue
    const int quarter = warp % 4;
    const uint32_t r = quarter * 32 + lane;
    const uint32_t r_row = r / a.box_w, r_col = r % a.box_w;
    uint32_t acc = 0, acc_phase = 0;
    for (uint32_t t = blockIdx.x; t < a.tiles; t += gridDim.x) {
      const uint32_t owt = t % a.ow_tiles;
      const uint32_t rest = t / a.ow_tiles;
      const uint32_t oh = (rest % a.oh_tiles) * a.rows + r_row;
      const uint32_t img = rest / a.oh_tiles;
      const uint32_t ow = owt * a.box_w + r_col;
      const bool valid = r < a.rows * a.box_w && ow < a.w_out && oh < a.h_out;
      const int64_t obase = valid ? static_cast<int64_t>(img) * a.co * a.hw + static_cast<int64_t>(oh) * a.w_out + ow : 0;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * N;
#pragma unroll 1
      for (int j0 = 0; j0 < N; j0 += 16) {
        uint32_t v[16];
        tmem_ld16(taddr + j0, v);
        if (valid) {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (j0 + q < static_cast<int>(a.co)) st_out(a.out + obase + static_cast<int64_t>(j0 + q) * a.hw, __uint_as_float(v[q]));
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
  if (warp == kProdWarps + 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

// packed[m][k] = F[m][k] (reference k order (c, fh, fw) = the filter's own layout), zero padded to Np x Kp.
template <bool BF16>
__global__ void pack_filter_direct_kernel(const float* __restrict__ flt, void* __restrict__ packed, int M, int K,
                                          int Np, int Kp) {
  const int64_t total = static_cast<int64_t>(Np) * Kp;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(i / Kp), k = static_cast<int>(i % Kp);
    const float v = (m < M && k < K) ? flt[static_cast<int64_t>(m) * K + k] : 0.0f;
    if constexpr (BF16) {
      reinterpret_cast<__nv_bfloat16*>(packed)[i] = __float2bfloat16_rn(v);
    } else {
      uint32_t r;
      asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(v));
      reinterpret_cast<uint32_t*>(packed)[i] = r;
    }
  }
}

}  // namespace tc
}  // namespace im2win

namespace {

struct DirectPlan {
  im2win::tc::DirectArgs a;
  int N, stages;
  size_t smem, packed_bytes;
};

// Fills `p` and returns true when the direct kernel applies to this problem.
bool plan_direct(int64_t n, int64_t c_in, int64_t h, int64_t w, int64_t c_out, int h_f, int w_f, int stride, int pad,
                 int bf16, DirectPlan& p) {
  using namespace im2win::tc;
  const char* env = getenv("IM2WIN_DIRECT");
  if (env && atoi(env) == 0) return false;
  if (c_in > 16 || c_out > 256 || pad < 0) return false;
  const int64_t hp = h + 2 * pad, wp = w + 2 * pad;
  if (h_f > hp || w_f > wp) return false;
  const int bk = bf16 ? 64 : 32;
  const int64_t K = c_in * h_f * w_f;
  const int64_t slabs = (K + bk - 1) / bk;
  p.N = c_out <= 64 ? 64 : c_out <= 96 ? 96 : c_out <= 128 ? 128 : 256;
  const int64_t h_out = (hp - h_f) / stride + 1, w_out = (wp - w_f) / stride + 1;
  DirectArgs& a = p.a;
  a = DirectArgs{};
  a.n_img = static_cast<uint32_t>(n);
  a.c_in = static_cast<uint32_t>(c_in);
  a.h_in = static_cast<uint32_t>(h);
  a.w_in = static_cast<uint32_t>(w);
  a.h_out = static_cast<uint32_t>(h_out);
  a.w_out = static_cast<uint32_t>(w_out);
  a.hw = static_cast<uint32_t>(h_out * w_out);
  a.co = static_cast<uint32_t>(c_out);
  a.stride = static_cast<uint32_t>(stride);
  a.h_f = static_cast<uint32_t>(h_f);
  a.w_f = static_cast<uint32_t>(w_f);
  a.pad = static_cast<uint32_t>(pad);
  if (w_out <= kTileM) {
    a.box_w = static_cast<uint32_t>(w_out);
    a.rows = static_cast<uint32_t>(std::min<int64_t>(h_out, kTileM / w_out));
  } else {
    const int64_t parts = (w_out + kTileM - 1) / kTileM;
    a.box_w = static_cast<uint32_t>((w_out + parts - 1) / parts);
    a.rows = 1;
  }
  a.ow_tiles = (a.w_out + a.box_w - 1) / a.box_w;
  a.oh_tiles = (a.h_out + a.rows - 1) / a.rows;
  const uint64_t tiles = static_cast<uint64_t>(n) * a.ow_tiles * a.oh_tiles;
  if (tiles >= (1ull << 32) || static_cast<uint64_t>(n) * h_out * w_out >= (1ull << 31) ||
      static_cast<uint64_t>(n) * c_in * h * w >= (1ull << 40))
    return false;
  a.tiles = static_cast<uint32_t>(tiles);
  a.K = static_cast<uint32_t>(K);
  a.slabs = static_cast<uint32_t>(slabs);
  a.kp = static_cast<uint32_t>(slabs * bk);
  a.prow = (a.rows - 1) * a.stride + a.h_f;
  a.pcol = (a.box_w - 1) * a.stride + a.w_f;
  a.pcolq = (a.pcol + a.stride - 1) / a.stride;
  a.prow_pitch = a.stride * a.pcolq;
  if (a.prow_pitch > 32u * kDirColIters) return false;
  // shared memory: A ring + resident filter + patch buffers
  const size_t b_bytes = static_cast<size_t>(slabs) * p.N * kRowBytes;
  const size_t patch_bytes = static_cast<size_t>(c_in) * a.prow * a.prow_pitch * 4;
  const size_t koff_bytes = (static_cast<size_t>(a.kp) * 4 + 15) & ~static_cast<size_t>(15);
  const size_t budget = 227 * 1024 - 2048;
  auto need = [&](int st, int pb) { return st * kTileM * kRowBytes + b_bytes + koff_bytes + pb * patch_bytes; };
  // deepest patch prefetch (up to 4 buffers) and A ring (2-4 stages) that fit
  p.stages = 4;
  a.patch_bufs = 4;
  if (const char* pb_env = getenv("IM2WIN_DIRECT_BUFS")) {  // A/B: patch buffers first, A stages to fit
    a.patch_bufs = static_cast<uint32_t>(std::min(4, std::max(1, atoi(pb_env))));
    while (need(p.stages, a.patch_bufs) > budget && p.stages > 2) --p.stages;
  }
  while (need(p.stages, a.patch_bufs) > budget && a.patch_bufs > 2) --a.patch_bufs;
  while (need(p.stages, a.patch_bufs) > budget && p.stages > 2) --p.stages;
  if (need(p.stages, a.patch_bufs) > budget) a.patch_bufs = 1;
  if (need(p.stages, a.patch_bufs) > budget) return false;
  p.smem = need(p.stages, a.patch_bufs) + 1024;
  p.packed_bytes = static_cast<size_t>(p.N) * a.kp * (bf16 ? 2 : 4);
  return true;
}

}  // namespace

int im2win_conv_direct_applies(int64_t n, int64_t c_in, int64_t h, int64_t w, int64_t c_out, int h_f, int w_f,
                               int stride, int pad, int bf16) {
  DirectPlan p;
  return plan_direct(n, c_in, h, w, c_out, h_f, w_f, stride, pad, bf16, p) ? 1 : 0;
}

size_t im2win_conv_direct_workspace_bytes(int64_t c_in, int64_t c_out, int h_f, int w_f, int bf16) {
  const int64_t bk = bf16 ? 64 : 32;
  const int64_t kp = (c_in * h_f * w_f + bk - 1) / bk * bk;
  return static_cast<size_t>(256 * kp * (bf16 ? 2 : 4)) + 256;
}

int im2win_launch_conv_tc_direct(const float* x, const float* flt, float* out, void* workspace, size_t ws_bytes,
                                 int64_t n, int64_t c_in, int64_t h, int64_t w, int64_t c_out, int h_f, int w_f,
                                 int stride, int pad, int bf16, cudaStream_t stream, const char** err) {
  using namespace im2win::tc;
  DirectPlan p;
  if (!plan_direct(n, c_in, h, w, c_out, h_f, w_f, stride, pad, bf16, p)) {
    *err = "im2win_conv_direct: shape not supported by the direct kernel (C <= 16, Co <= 256, window fits smem)";
    return 1;
  }
  if (ws_bytes < p.packed_bytes) {
    *err = "im2win_conv_direct: workspace too small";
    return 1;
  }
  DirectArgs a = p.a;
  a.x = x;
  a.bpk = workspace;
  a.out = out;
  const int N = p.N;
  if (bf16)
    pack_filter_direct_kernel<true><<<256, 256, 0, stream>>>(flt, workspace, static_cast<int>(c_out),
                                                             static_cast<int>(a.K), N, static_cast<int>(a.kp));
  else
    pack_filter_direct_kernel<false><<<256, 256, 0, stream>>>(flt, workspace, static_cast<int>(c_out),
                                                              static_cast<int>(a.K), N, static_cast<int>(a.kp));
  const size_t smem = p.smem;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t grid = a.tiles < static_cast<uint32_t>(sms) ? a.tiles : static_cast<uint32_t>(sms);
  cudaError_t e = cudaSuccess;
#define IM2WIN_DIR(BF, NN, ST)                                                                          \
  {                                                                                                     \
    auto kern = conv_tc_direct_kernel<BF, NN, ST>;                                                      \
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)); \
    if (e == cudaSuccess) {                                                                             \
      im2win_note_kernel(BF ? "conv_tc_direct_kernel (in-SM im2win windows, bf16)"                      \
                            : "conv_tc_direct_kernel (in-SM im2win windows, tf32)");                    \
      kern<<<grid, kDirThreads, smem, stream>>>(a);                                                     \
      e = cudaGetLastError();                                                                           \
    }                                                                                                   \
  }
#define IM2WIN_DIR_N(BF, ST)                       \
  switch (N) {                                     \
    case 64: IM2WIN_DIR(BF, 64, ST) break;         \
    case 96: IM2WIN_DIR(BF, 96, ST) break;         \
    case 128: IM2WIN_DIR(BF, 128, ST) break;       \
    default: IM2WIN_DIR(BF, 256, ST) break;        \
  }
  const int stages = p.stages;
  if (bf16) {
    if (stages >= 4) { IM2WIN_DIR_N(true, 4) } else if (stages == 3) { IM2WIN_DIR_N(true, 3) } else { IM2WIN_DIR_N(true, 2) }
  } else {
    if (stages >= 4) { IM2WIN_DIR_N(false, 4) } else if (stages == 3) { IM2WIN_DIR_N(false, 3) } else { IM2WIN_DIR_N(false, 2) }
  }
#undef IM2WIN_DIR_N
#undef IM2WIN_DIR
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 2;
  }
  return 0;
}
