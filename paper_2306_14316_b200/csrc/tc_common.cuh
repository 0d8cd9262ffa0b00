// tcgen05 / TMEM / TMA / mbarrier helpers shared by the tensor-core kernels (sm_100a).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

#include "common.cuh"

namespace im2win {
namespace tc {

constexpr int kTileM = 128;        // pixels per tile (UMMA M)
constexpr int kRowBytes = 128;     // one swizzle-128B row of K per stage
// TMA-fed kernels: warp 0 TMA, warp 1 MMA, warp 2 TMEM allocator, warp 3 idle,
// warps 4..4+kEpiWarps-1 epilogue (two warps per TMEM lane quarter, one per column half).
constexpr int kEpiWarps = 8;
constexpr int kTcThreads = (4 + kEpiWarps) * 32;

// ---------------------------------------------------------------- PTX helpers
IM2WIN_DEVICE void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
IM2WIN_DEVICE void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
IM2WIN_DEVICE void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
IM2WIN_DEVICE void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
IM2WIN_DEVICE void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
IM2WIN_DEVICE void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
IM2WIN_DEVICE void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
IM2WIN_DEVICE void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

IM2WIN_DEVICE void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

IM2WIN_DEVICE uint64_t smem_desc_sw128(uint32_t addr) {
  // K-major, 128-byte swizzle: 8-row atoms of 1024 B (SBO), LBO unused (=16 B), version 1 (sm_100)
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// K-major, 64-byte swizzle (rows of 64 B): 8-row atoms of 512 B (SBO), layout type 4 (sm_100)
IM2WIN_DEVICE uint64_t smem_desc_sw64(uint32_t addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(512 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(4) << 61;
  return d;
}
template <int ROW>
IM2WIN_DEVICE uint64_t smem_desc_row(uint32_t addr) {
  if constexpr (ROW == 64) return smem_desc_sw64(addr);
  else return smem_desc_sw128(addr);
}

template <bool BF16, int N>
__host__ __device__ constexpr uint32_t instr_desc() {
  // c_format F32 (bit 4), a/b format (bits 7-9 / 10-12: BF16=1, TF32=2), K-major A and B,
  // n_dim = N>>3 (bits 17-22), m_dim = M>>4 (bits 24-28)
  return (1u << 4) | ((BF16 ? 1u : 2u) << 7) | ((BF16 ? 1u : 2u) << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(kTileM >> 4) << 24);
}

template <bool BF16>
IM2WIN_DEVICE void mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  if constexpr (BF16) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  }
}

// Warp-converged MMA issue: the whole warp runs the issue loop (descriptors and loop state stay
// warp-uniform, so they live in uniform registers) and elect.sync picks the one issuing lane.
// With the loop inside `if (lane == 0)` ptxas wraps every UTCHMMA in an elect loop and moves the
// descriptors through R2UR (measured: phase kernel conv4 10% slower).
template <bool BF16, bool PAIR = false>
IM2WIN_DEVICE void mma_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
#define IM2WIN_MMA_WARP(GROUP, KIND)                                                                     \
  asm volatile(                                                                                          \
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"             \
      "@e tcgen05.mma.cta_group::" GROUP ".kind::" KIND " [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),  \
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate))
  if constexpr (PAIR && BF16) IM2WIN_MMA_WARP("2", "f16");
  else if constexpr (PAIR) IM2WIN_MMA_WARP("2", "tf32");
  else if constexpr (BF16) IM2WIN_MMA_WARP("1", "f16");
  else IM2WIN_MMA_WARP("1", "tf32");
#undef IM2WIN_MMA_WARP
}
template <bool PAIR = false>
IM2WIN_DEVICE void mma_commit_warp(uint64_t* bar) {
  if constexpr (PAIR) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n"
        ::"r"(smem_u32(bar)), "h"(static_cast<uint16_t>(3))
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
            smem_u32(bar))
        : "memory");
  }
}

IM2WIN_DEVICE void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

// ---------------------------------------------------------------- CTA pairs (cta_group::2)
// Two CTAs of a 2-CTA cluster run one UMMA of M = 256: each holds its own 128 A rows and half
// of the B rows in shared memory at the same offsets; the accumulator rows of CTA r live in its
// own TMEM.  Only the even CTA (rank 0) issues MMAs; TMA loads of both CTAs signal rank 0's
// full barrier; MMA completion is multicast to the barriers of both CTAs.
IM2WIN_DEVICE uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
// shared::cluster address of this CTA's shared variable `p` in cluster CTA `rank`
IM2WIN_DEVICE uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(d) : "r"(smem_u32(p)), "r"(rank));
  return d;
}
IM2WIN_DEVICE void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
IM2WIN_DEVICE void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
template <bool BF16>
IM2WIN_DEVICE void mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  if constexpr (BF16) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  }
}
// arrive on barrier `bar` (same offset) of both CTAs of the pair when this thread's MMAs complete
IM2WIN_DEVICE void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
template <bool BF16, int N, int M>
__host__ __device__ constexpr uint32_t instr_desc_m() {
  return (1u << 4) | ((BF16 ? 1u : 2u) << 7) | ((BF16 ? 1u : 2u) << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

IM2WIN_DEVICE void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// Output store of the TC epilogues (lane = pixel: one 128-byte piece of a channel plane per warp
// instruction).  IM2WIN_ST_MODE (build flag, A/B with tools/lib_ab.py): 0 plain st.global,
// 1 st.global.cs (streaming; default), 2 L2::evict_last policy, 3 L2::evict_first policy,
// 4 st.global.wt.  Measured (N=128, production path): .cs +1-4% on conv9/conv10 BF16, else
// within 1%; evict_last +5% on conv7 but -10% on conv8 BF16; evict_first -1..-10%.
#ifndef IM2WIN_ST_MODE
#define IM2WIN_ST_MODE 1
#endif
IM2WIN_DEVICE void st_out(float* p, float v) {
#if IM2WIN_ST_MODE == 9  // exploration: no output stores (wrong results; times the rest of the kernel)
  if (__float_as_uint(v) == 0x7fffffffu) *p = v;
#elif IM2WIN_ST_MODE == 1
  __stcs(p, v);
#elif IM2WIN_ST_MODE == 2 || IM2WIN_ST_MODE == 3
  uint64_t pol;
#if IM2WIN_ST_MODE == 2
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
#else
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
#endif
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;\n" ::"l"(p), "f"(v), "l"(pol) : "memory");
#elif IM2WIN_ST_MODE == 4
  __stwt(p, v);
#else
  *p = v;
#endif
}

IM2WIN_DEVICE uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return r;
}

IM2WIN_DEVICE uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}


IM2WIN_DEVICE void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// ---------------------------------------------------------------- in-kernel channels-last feed
// The TMA-fed kernels read a channels-last copy Xcl of the NCHW input.  Written by a separate
// kernel, that copy costs a full HBM pass (0.42 of conv4's 1.17 ms in BF16) in series with
// the conv.  With a feed, kFeedWarps extra warps per CTA of the conv kernel itself produce Xcl
// while the tensor cores work: blocks of units of (image, channel group, pixel chunk) are dealt
// to the feed warps of all CTAs round-robin, so the copy advances image by image in the order
// the conv consumes it; each finished block bumps its image's ready counter with release
// semantics.  The TMA producer waits
// (acquire) for every image its next tile reads before issuing the loads.  CTAs wait on each
// other, so the kernel is launched cooperatively (all CTAs co-resident, or no launch).
// The ready counters are zeroed by the host before the launch (cudaMemsetAsync).
constexpr int kFeedWarps = 8;
#ifndef IM2WIN_TC_BOUND_THREADS
constexpr int kTcThreadsFeed = kTcThreads + 32 * kFeedWarps;
#else  // exploration builds: launch bounds of the non-feed kernel (the feed then cannot launch)
constexpr int kTcThreadsFeed = IM2WIN_TC_BOUND_THREADS;
#endif

// A unit: G channels (one 32-byte run of Xcl per pixel) x 32*J pixels; each lane loads
// G*J values (one coalesced 128-byte row per channel and j) before storing any.
template <bool BF16>
struct FeedShape {
  static constexpr uint32_t G = BF16 ? 16 : 8;
  static constexpr uint32_t J = BF16 ? 2 : 4;
  static constexpr uint32_t kPix = 32 * J;
};

struct NhwcFeed {
  const float* src;        // NCHW float32 input; nullptr: Xcl already exists, no feed
  void* dst;               // Xcl [n][h*w][c_pad] (bf16 or f32)
  uint32_t c_in, c_pad, hw, n_img;
  uint32_t chunks;         // ceil(hw / kPix)
  uint32_t units_per_img;  // chunks * ceil(c_pad / G)
  uint32_t* ready;         // [n_img] finished units per image
  uint32_t* front;         // highest image any TMA producer has started a tile of
  uint32_t lookahead;      // the feed converts image i only once front >= i - lookahead
  uint32_t nowait;         // A/B probe only (IM2WIN_FEED_NOWAIT): the producer does not wait
};

// Throttle: keep the channels-last copy at most `lookahead` images ahead of the conv, so the
// bytes the feed writes are still in L2 when the TMA engine reads them (a feed running far
// ahead pushes its copy to HBM and competes with the conv for bandwidth).  lookahead is at
// least one grid-round of images (set by the launcher), so no producer waits on a throttled unit.
IM2WIN_DEVICE void feed_throttle(const NhwcFeed& f, uint32_t img) {
  for (;;) {
    uint32_t fr;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(fr) : "l"(f.front) : "memory");
    if (img <= fr || img - fr <= f.lookahead) return;
    __nanosleep(256);
  }
}

IM2WIN_DEVICE void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }

// One converter warp: blocks of kFeedBatch consecutive units (one image, mostly), dealt
// round-robin.  Two units are in flight: the loads of unit i+1 are issued before unit i is
// converted and stored.  The ready counter is bumped (after a fence) at the end of a block or
// where a block crosses into the next image -- one fence round trip per block, not per unit.
constexpr uint32_t kFeedBatch = 8;

template <bool BF16>
IM2WIN_DEVICE void feed_load(const NhwcFeed& f, uint32_t u, int lane, float (&v)[FeedShape<BF16>::J][FeedShape<BF16>::G]) {
  using S = FeedShape<BF16>;
  const uint32_t img = u / f.units_per_img;
  const uint32_t r = u - img * f.units_per_img;
  const uint32_t cg = (r / f.chunks) * S::G;
  const uint32_t p0 = (r % f.chunks) * S::kPix;
  const float* s = f.src + static_cast<uint64_t>(img) * f.c_in * f.hw;
#pragma unroll
  for (uint32_t c = 0; c < S::G; ++c)
#pragma unroll
    for (uint32_t j = 0; j < S::J; ++j) {
      const uint32_t p = p0 + j * 32 + lane, ch = cg + c;
      v[j][c] = (ch < f.c_in && p < f.hw) ? __ldcs(s + static_cast<uint64_t>(ch) * f.hw + p) : 0.0f;
    }
}

template <bool BF16>
IM2WIN_DEVICE void feed_store(const NhwcFeed& f, uint32_t u, int lane,
                              const float (&v)[FeedShape<BF16>::J][FeedShape<BF16>::G]) {
  using S = FeedShape<BF16>;
  constexpr uint32_t kGran = BF16 ? 8 : 4;  // channels per 16-byte store
  const uint32_t img = u / f.units_per_img;
  const uint32_t r = u - img * f.units_per_img;
  const uint32_t cg = (r / f.chunks) * S::G;
  const uint32_t p0 = (r % f.chunks) * S::kPix;
  const uint32_t grans = min(S::G, f.c_pad - cg) / kGran;
#pragma unroll
  for (uint32_t j = 0; j < S::J; ++j) {
    const uint32_t p = p0 + j * 32 + lane;
    if (p >= f.hw) continue;
    const uint64_t o = (static_cast<uint64_t>(img) * f.hw + p) * f.c_pad + cg;
#pragma unroll
    for (uint32_t g = 0; g < S::G / kGran; ++g) {
      if (g >= grans) break;
      if constexpr (BF16) {
        uint4 q;
        q.x = pack_bf16x2(v[j][8 * g], v[j][8 * g + 1]);
        q.y = pack_bf16x2(v[j][8 * g + 2], v[j][8 * g + 3]);
        q.z = pack_bf16x2(v[j][8 * g + 4], v[j][8 * g + 5]);
        q.w = pack_bf16x2(v[j][8 * g + 6], v[j][8 * g + 7]);
        *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(f.dst) + o + 8 * g) = q;
      } else {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(f.dst) + o + 4 * g) =
            make_float4(v[j][4 * g], v[j][4 * g + 1], v[j][4 * g + 2], v[j][4 * g + 3]);
      }
    }
  }
}

// Publish `count` finished units of image `img`: the TMA engine (async proxy) of another SM
// reads these bytes next.
IM2WIN_DEVICE void feed_publish(const NhwcFeed& f, uint32_t img, uint32_t count, int lane) {
  fence_proxy_async_global();
  __syncwarp();
  if (lane == 0)
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(f.ready + img), "r"(count) : "memory");
  __syncwarp();
}

template <bool BF16>
IM2WIN_DEVICE void nhwc_feed_run(const NhwcFeed& f, int lane, uint32_t feed_warp, uint32_t feed_warps) {
  using S = FeedShape<BF16>;
  const uint32_t total = f.n_img * f.units_per_img;
  // this warp's units: blocks of kFeedBatch consecutive units, every feed_warps-th block
  auto step = [&](uint32_t u) { return (u + 1) % kFeedBatch ? u + 1 : u + 1 + (feed_warps - 1) * kFeedBatch; };
  auto may_load = [&](uint32_t u) {  // the throttle would not hold unit u back
    uint32_t fr;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(fr) : "l"(f.front) : "memory");
    const uint32_t img = u / f.units_per_img;
    return img <= fr || img - fr <= f.lookahead;
  };
  float va[S::J][S::G], vb[S::J][S::G];
  uint32_t pend_img = 0, pend = 0;
  auto publish = [&]() {
    if (pend) feed_publish(f, pend_img, pend, lane);
    pend = 0;
  };
  // store unit u (data v) and account for it; publish at image changes and block ends
  auto finish = [&](uint32_t u, uint32_t next, const float(&v)[S::J][S::G]) {
    const uint32_t img = u / f.units_per_img;
    if (pend && img != pend_img) publish();
    feed_store<BF16>(f, u, lane, v);
    pend_img = img;
    ++pend;
    if (next != u + 1) publish();
  };
  // The next unit's loads are issued before the current unit is stored -- unless the throttle
  // would hold it: then the current unit is stored and published first (the conv may be
  // waiting for it), and only then does the warp wait.
  uint32_t ua = feed_warp * kFeedBatch;
  if (ua < total) {
    feed_throttle(f, ua / f.units_per_img);
    feed_load<BF16>(f, ua, lane, va);
  }
  while (ua < total) {
    const uint32_t ub = step(ua);
    bool pre = ub < total && may_load(ub);
    if (pre) feed_load<BF16>(f, ub, lane, vb);
    finish(ua, ub, va);
    if (ub >= total) break;
    if (!pre) {
      publish();
      feed_throttle(f, ub / f.units_per_img);
      feed_load<BF16>(f, ub, lane, vb);
    }
    const uint32_t uc = step(ub);
    pre = uc < total && may_load(uc);
    if (pre) feed_load<BF16>(f, uc, lane, va);
    finish(ub, uc, vb);
    if (uc >= total) break;
    if (!pre) {
      publish();
      feed_throttle(f, uc / f.units_per_img);
      feed_load<BF16>(f, uc, lane, va);
    }
    ua = uc;
  }
  publish();
}

// Producer side: block until images [lo, hi] are complete.  [conf_lo, conf_hi] caches the
// last confirmed contiguous range (tiles arrive in increasing image order per CTA).
IM2WIN_DEVICE void nhwc_feed_wait(const NhwcFeed& f, uint32_t lo, uint32_t hi, uint32_t& conf_lo,
                                  uint32_t& conf_hi) {
  if (f.src == nullptr || f.nowait) return;
  if (hi >= f.n_img) hi = f.n_img - 1;
  // publish the conv front (the feed's throttle); once per new highest image
  if (!(conf_lo <= conf_hi && hi <= conf_hi)) atomicMax(f.front, hi);
  bool waited = false;
  for (uint32_t i = lo; i <= hi; ++i) {
    if (i >= conf_lo && i <= conf_hi) continue;
    uint32_t v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(f.ready + i) : "memory");
      if (v >= f.units_per_img) break;
      __nanosleep(64);
    }
    waited = true;
    if (conf_hi + 1 == i && conf_lo <= conf_hi) conf_hi = i;
    else { conf_lo = i; conf_hi = i; }
  }
  if (waited) fence_proxy_async_global();
}

// Feed lookahead for a persistent grid walking `items` work items over n_img images in image
// order: one grid-round of images plus two (the producers of a round never wait on a throttled unit).
inline NhwcFeed feed_for(const NhwcFeed& f, uint64_t grid, uint64_t items) {
  NhwcFeed g = f;
  // IM2WIN_FEED_ROUNDS: lookahead in grid-rounds (A/B; 0 = unthrottled)
  static const int rounds = getenv("IM2WIN_FEED_ROUNDS") ? atoi(getenv("IM2WIN_FEED_ROUNDS")) : 0;
  if (g.src && items) {
    g.lookahead = rounds <= 0 ? 0xffffffffu
                              : static_cast<uint32_t>(rounds * ((grid * g.n_img + items - 1) / items) + 2);
  }
  return g;
}

// Launch of a TMA-fed conv kernel: with a feed, the extra converter warps and a cooperative
// launch (the CTAs wait on each other's feed units, so all must be co-resident).
// cluster = 2: CTA pairs (cta_group::2 kernels).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_tc_kernel(void (*kern)(KArgs...), uint32_t grid, size_t smem, cudaStream_t stream,
                                    bool feed, int cluster, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(feed ? kTcThreadsFeed : kTcThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (feed) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  if (cluster > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Largest number of co-resident 2-CTA clusters for a kernel configuration (0 on error).
template <typename... KArgs>
inline int max_pair_clusters(void (*kern)(KArgs...), size_t smem, bool feed) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(feed ? kTcThreadsFeed : kTcThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

inline PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace tc
}  // namespace im2win
