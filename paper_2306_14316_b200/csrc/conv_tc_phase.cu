// Phase-shift tensor-core convolution: the im2win window reuse for any stride, two
// pixel tiles per CTA work item.
//
// im2win stores each output row's windows so that consecutive windows overlap
// (layouts.py:73-83; test_layouts.py:187-199).  With stride s, filter tap fw = s*q + r
// (phase r < s, shift q) reads input column s*(ow + q) + r, so the A tile of tap fw is
// the phase-r column sequence P_r[j] = X[.., s*j + r, :] shifted by q rows.  One TMA box
// per (fh, phase, channel chunk) therefore feeds all ceil((Wf - r)/s) taps of that phase
// through smem descriptors advanced by q rows (q * 128 B): A is fetched Wf/s times less
// often than by the generic fused kernel (conv_tc_fused.cu), which fetches it per tap.
// Each work item holds MT = 2 or 4 pixel tiles (MT UMMA M=128 accumulators in TMEM) so every
// staged filter tile feeds MT MMAs: filter traffic from L2 drops by MT as well.
//
//   A map (one per phase r): {c, j, fh % s, (oh*s + fh) / s, n} over the channels-last
//     copy Xcl, strides {1, s*C, W*C, s*W*C, H*W*C} elements, base Xcl + r*C;
//     box {BK, pitch, 1, rows, box_n}, pitch = box_w + qmax, qmax = (Wf - 1) / s.
//   B: the packed filter B[m][(fh*Wf + fw)*Kc + c] (pack_filter_shift_kernel).
//   K loop: fh, phase r, channel chunk -> nq(r) taps x BK/UK MMAs x MT tiles.
// D rows whose column position in the pitch is >= box_w are padding and are not stored.
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "tc_common.cuh"

namespace im2win {
namespace tc {

struct PhaseArgs {
  float* __restrict__ out;
  uint32_t n_img, h_out, w_out, hw, co;
  uint32_t box_w, pitch, rows, box_n;  // pixel tile: box_n images x rows output rows x box_w columns
  uint32_t ow_tiles, oh_tiles, n_tiles, p_tiles, pairs, co_tiles;
  uint32_t stride, w_f, c_slabs, k_iters;  // k_iters = Hf * stride * c_slabs
  uint32_t k_total;                        // Kp of the packed filter (a box there is all zero fill)
};

constexpr int kPhRows = 136;  // 128 MMA rows + up to 8 rows of shift

// PAIR: a 2-CTA cluster runs UMMA M = 256 (cta_group::2): each CTA stages its own MT pixel
// tiles and half of each filter tap (N/2 rows), so the per-SM shared-memory operand bytes per
// MMA drop from (128 + N) to (128 + N/2) rows and the filter's L2->SM traffic halves.  Work
// items are then 2*MT pixel tiles (MT per CTA).  Rank 0 issues the MMAs.
// TN2: two taps per MMA (Co <= 64): B rows 0-63 are tap q, rows 64-127 tap q+1 -- the ring's
// consecutive tap tiles -- both against the A tile shifted for tap q, so D columns 64-127 hold
// tap q+1 one pixel early and the epilogue adds D[p][co] + D[p+1][64+co].  A 128x128x16 UMMA
// reads 8 KB of operands for twice the work of a 128x64x16 one (6 KB): 64 vs 2 x 48 cycles
// (tools/probes/umma_rate.cu).  An odd last tap runs as a plain N=64 MMA into columns 0-63.
template <bool BF16, int N, int STAGES, int TAPS, int MT, bool PAIR, bool TN2 = false>
__global__ void __launch_bounds__(kTcThreadsFeed, 1)
    conv_tc_phase_kernel(const PhaseArgs a, const __grid_constant__ CUtensorMap tmap_a0,
                         const __grid_constant__ CUtensorMap tmap_a1, const __grid_constant__ CUtensorMap tmap_b,
                         const NhwcFeed feed) {
  constexpr uint32_t kATile = kPhRows * kRowBytes;  // 17 KB, multiple of 1024
  constexpr uint32_t kABytes = MT * kATile;
  // PAIR && TN2: a pair MMA is M=256 x N=128 -- CTA rank r holds tap 2j + r of pair j (all 64
  // filter rows), so each CTA stages ceil(TAPS/2) tap tiles and B's halves are the two taps
  constexpr bool kPT = PAIR && TN2;
  constexpr int kBRows = PAIR && !TN2 ? N / 2 : N;  // filter rows per staged tile
  constexpr int kBSlots = kPT ? (TAPS + 1) / 2 : TAPS;
  constexpr uint32_t kBTap = kBRows * kRowBytes;
  constexpr uint32_t kStageBytes = kABytes + kBSlots * kBTap;
  constexpr int kBK = BF16 ? 64 : 32;
  constexpr int kUK = BF16 ? 16 : 8;
  constexpr int kAccN = TN2 ? 2 * N : N;  // TMEM columns per pixel tile
  constexpr uint32_t kTmemCols = (2 * MT * kAccN <= 128) ? 128 : (2 * MT * kAccN <= 256 ? 256 : 512);
  constexpr uint32_t kIdesc = instr_desc_m<BF16, N, PAIR ? 256 : 128>();
  constexpr uint32_t kIdesc2 = instr_desc_m<BF16, 2 * N, PAIR ? 256 : 128>();
  static_assert(!TN2 || N == 64, "tap pairs: Co tile 64");
  constexpr uint32_t kCtas = PAIR ? 2 : 1;
  static_assert(kATile % 1024 == 0 && kBTap % 1024 == 0, "tiles must keep 1024 B alignment");
  static_assert(2 * MT * kAccN <= 512, "TMEM holds 512 fp32 columns");

  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[2];
  __shared__ __align__(8) uint64_t tempty_bar[2];
  __shared__ uint32_t tmem_base_sh;
  // TN2: each quarter warp's first-row tap-(q+1) columns, for the warp of the quarter before it
  __shared__ float xch[TN2 ? 2 * MT * 2 * 4 * 32 : 1];

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t loaded_rows = a.pitch * a.rows * a.box_n;
  const uint32_t a_box_bytes = loaded_rows * kRowBytes;
  const uint32_t s = a.stride;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  // work items walk per CTA (or per CTA pair): t = blockIdx.x [/ 2] + k * gridDim.x [/ 2], written
  // out at each loop -- a hoisted unit/units pair made ptxas move the MMA warp's descriptor math
  // from uniform to regular registers (R2UR per MMA; conv4 10% slower)

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], kCtas * kEpiWarps);
    }
    fence_barrier_init();
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmap_a0) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmap_a1) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmap_b) : "memory");
  }
  if (warp == 2) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                       smem_u32(&tmem_base_sh)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                       smem_u32(&tmem_base_sh)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
  }
  // rows past the TMA box feed only padding D rows; keep them finite
  for (uint32_t i = threadIdx.x; i < STAGES * kStageBytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // the peer's barriers are initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;
  const uint32_t total = a.pairs * a.co_tiles;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      uint32_t conf_lo = 1, conf_hi = 0;
      for (uint32_t t = PAIR ? blockIdx.x / 2 : blockIdx.x; t < total; t += PAIR ? gridDim.x / 2 : gridDim.x) {
        const uint32_t co_blk = t % a.co_tiles;
        const uint32_t pair = t / a.co_tiles;
        uint32_t ow0[MT], oh0[MT], n0[MT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          // past the last pixel tile: coordinates past the tensor (TMA zero-fills), D not stored
          uint32_t pt = (PAIR ? pair * 2 + rank : pair) * MT + mt;
          ow0[mt] = (pt % a.ow_tiles) * a.box_w;
          pt /= a.ow_tiles;
          oh0[mt] = (pt % a.oh_tiles) * a.rows;
          n0[mt] = (pt / a.oh_tiles) * a.box_n;
        }
        // pixel tiles are image-major: n0[0] is the lowest image, n0[MT-1] the highest
        nhwc_feed_wait(feed, n0[0], n0[MT - 1] + a.box_n - 1, conf_lo, conf_hi);
        for (uint32_t ki = 0; ki < a.k_iters; ++ki) {
          const uint32_t c0 = (ki % a.c_slabs) * kBK;
          const uint32_t rem = ki / a.c_slabs;
          const uint32_t r = rem % s, fh = rem / s;
          const uint32_t nq = (a.w_f - r + s - 1) / s;
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * kStageBytes;
          const CUtensorMap* am = r == 0 ? &tmap_a0 : &tmap_a1;
          if constexpr (kPT) {
            // pair j: this CTA stages tap 2j + rank (a tap past the phase's last is a box beyond the
            // packed filter's K extent: zero-filled, so its half of the MMA adds nothing)
            const uint32_t slots = (nq + 1) / 2;
            if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * (MT * a_box_bytes + slots * kBTap));
            const uint32_t fb = mapa_shared(&full_bar[stage], 0);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              asm volatile(
                  "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
                  "[%1, {%3, %4, %5, %6, %7}], [%2];\n" ::"r"(smem_u32(st + mt * kATile)),
                  "l"(am), "r"(fb), "r"(c0), "r"(ow0[mt]), "r"(fh % s), "r"(oh0[mt] + fh / s), "r"(n0[mt])
                  : "memory");
            }
            for (uint32_t j = 0; j < slots; ++j) {
              const uint32_t q = 2 * j + rank;
              const uint32_t kx = q < nq ? (fh * a.w_f + s * q + r) * a.c_slabs * kBK + c0 : a.k_total;
              asm volatile(
                  "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
                  "[%1, {%3, %4}], [%2];\n" ::"r"(smem_u32(st + kABytes + j * kBTap)),
                  "l"(&tmap_b), "r"(fb), "r"(kx), "r"(co_blk * N)
                  : "memory");
            }
          } else if constexpr (PAIR) {
            // both CTAs' loads complete on rank 0's full barrier, which expects the bytes of both
            if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * (MT * a_box_bytes + nq * kBTap));
            const uint32_t fb = mapa_shared(&full_bar[stage], 0);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              asm volatile(
                  "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
                  "[%1, {%3, %4, %5, %6, %7}], [%2];\n" ::"r"(smem_u32(st + mt * kATile)),
                  "l"(am), "r"(fb), "r"(c0), "r"(ow0[mt]), "r"(fh % s), "r"(oh0[mt] + fh / s), "r"(n0[mt])
                  : "memory");
            }
            for (uint32_t q = 0; q < nq; ++q)
              asm volatile(
                  "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
                  "[%1, {%3, %4}], [%2];\n" ::"r"(smem_u32(st + kABytes + q * kBTap)),
                  "l"(&tmap_b), "r"(fb), "r"((fh * a.w_f + s * q + r) * a.c_slabs * kBK + c0),
                  "r"(co_blk * N + rank * kBRows)
                  : "memory");
          } else {
            mbar_arrive_expect_tx(&full_bar[stage], MT * a_box_bytes + nq * kBTap);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              asm volatile(
                  "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
                  "%5, %6, %7}], [%2];\n" ::"r"(smem_u32(st + mt * kATile)),
                  "l"(am), "r"(smem_u32(&full_bar[stage])), "r"(c0), "r"(ow0[mt]), "r"(fh % s),
                  "r"(oh0[mt] + fh / s), "r"(n0[mt])
                  : "memory");
            }
            for (uint32_t q = 0; q < nq; ++q)
              tma_load_2d(st + kABytes + q * kBTap, &tmap_b, &full_bar[stage],
                          (fh * a.w_f + s * q + r) * a.c_slabs * kBK + c0, co_blk * N);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if constexpr (!PAIR) {
      // (the single-lane issue loop exactly as before the pair variant: ptxas keeps its descriptor
      // arithmetic in uniform registers; variants of it measured 10% slower on conv4)
      if (lane == 0) {
        uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
        for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
          mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t tmem_d = tmem_base + acc * (MT * kAccN);
          for (uint32_t ki = 0; ki < a.k_iters; ++ki) {
            const uint32_t r = (ki / a.c_slabs) % s;
            const uint32_t nq = (a.w_f - r + s - 1) / s;
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            const uint32_t abase = smem_u32(smem + stage * kStageBytes);
            const uint32_t bbase = abase + kABytes;
            if constexpr (TN2) {
#pragma unroll
              for (int q = 0; q < TAPS; q += 2) {
                if (q + 1 < static_cast<int>(nq)) {
#pragma unroll
                  for (int kk = 0; kk < kBK / kUK; ++kk) {
                    const uint64_t bd = smem_desc_sw128(bbase + q * kBTap + kk * 32);  // taps q, q+1: 128 rows
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt)
                      mma<BF16>(tmem_d + mt * kAccN, smem_desc_sw128(abase + mt * kATile + q * kRowBytes + kk * 32),
                                bd, kIdesc2, (ki | q | kk) != 0);
                  }
                } else if (q < static_cast<int>(nq)) {
#pragma unroll
                  for (int kk = 0; kk < kBK / kUK; ++kk) {
                    const uint64_t bd = smem_desc_sw128(bbase + q * kBTap + kk * 32);
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt)
                      mma<BF16>(tmem_d + mt * kAccN, smem_desc_sw128(abase + mt * kATile + q * kRowBytes + kk * 32),
                                bd, kIdesc, (ki | q | kk) != 0);
                  }
                }
              }
              mma_commit(&empty_bar[stage]);
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
              continue;
            }
#pragma unroll
            for (int q = 0; q < TAPS; ++q) {
              if (q < static_cast<int>(nq)) {
#pragma unroll
                for (int kk = 0; kk < kBK / kUK; ++kk) {
                  const uint64_t bd = smem_desc_sw128(bbase + q * kBTap + kk * 32);
#pragma unroll
                  for (int mt = 0; mt < MT; ++mt)
#ifdef IM2WIN_PHASE_NOSHIFT  // exploration builds only: wrong results, times an unshifted A read
                    mma<BF16>(tmem_d + mt * N, smem_desc_sw128(abase + mt * kATile + kk * 32), bd, kIdesc,
                              (ki | q | kk) != 0);
#else
                    mma<BF16>(tmem_d + mt * N, smem_desc_sw128(abase + mt * kATile + q * kRowBytes + kk * 32), bd,
                              kIdesc, (ki | q | kk) != 0);
#endif
                }
              }
            }
            mma_commit(&empty_bar[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          mma_commit(&tfull_bar[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      }
    } else if (lane == 0 && rank == 0) {
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      for (uint32_t t = PAIR ? blockIdx.x / 2 : blockIdx.x; t < total; t += PAIR ? gridDim.x / 2 : gridDim.x) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * (MT * kAccN);
        for (uint32_t ki = 0; ki < a.k_iters; ++ki) {
          const uint32_t r = (ki / a.c_slabs) % s;
          const uint32_t nq = (a.w_f - r + s - 1) / s;
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t abase = smem_u32(smem + stage * kStageBytes);
          const uint32_t bbase = abase + kABytes;
          if constexpr (kPT) {
#pragma unroll
            for (int j = 0; j < kBSlots; ++j) {
              if (2 * j < static_cast<int>(nq)) {
#pragma unroll
                for (int kk = 0; kk < kBK / kUK; ++kk) {
                  const uint64_t bd = smem_desc_sw128(bbase + j * kBTap + kk * 32);
#pragma unroll
                  for (int mt = 0; mt < MT; ++mt)
                    mma_pair<BF16>(tmem_d + mt * kAccN,
                                   smem_desc_sw128(abase + mt * kATile + 2 * j * kRowBytes + kk * 32), bd, kIdesc2,
                                   (ki | j | kk) != 0);
                }
              }
            }
            mma_commit_pair(&empty_bar[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
#pragma unroll
          for (int q = 0; q < TAPS; ++q) {
            if (q < static_cast<int>(nq)) {
#pragma unroll
              for (int kk = 0; kk < kBK / kUK; ++kk) {
                const uint64_t bd = smem_desc_sw128(bbase + q * kBTap + kk * 32);
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
                  mma_pair<BF16>(tmem_d + mt * N, smem_desc_sw128(abase + mt * kATile + q * kRowBytes + kk * 32), bd,
                                 kIdesc, (ki | q | kk) != 0);
              }
            }
          }
          mma_commit_pair(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit_pair(&tfull_bar[acc]);
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
    const uint32_t rr = quarter * 32 + lane;
    const uint32_t per_img = a.pitch * a.rows;
    const uint32_t r_n = rr / per_img, r_rem = rr % per_img;
    const uint32_t r_h = r_rem / a.pitch, r_w = r_rem % a.pitch;
    uint32_t acc = 0, acc_phase = 0;
    for (uint32_t t = PAIR ? blockIdx.x / 2 : blockIdx.x; t < total; t += PAIR ? gridDim.x / 2 : gridDim.x) {
      const uint32_t co_blk = t % a.co_tiles;
      const uint32_t pair = t / a.co_tiles;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
#ifndef IM2WIN_PHASE_EPI_TILEMAJOR
      // the MT tiles' pieces of each channel plane are stored back to back (consecutive output
      // rows of a plane: longer DRAM write runs, tools/probes/nchw_store_probe.cu)
      int64_t obase[MT];
      bool valid[MT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        uint32_t pt = (PAIR ? pair * 2 + rank : pair) * MT + mt;
        const bool tile_ok = pt < a.p_tiles;
        const uint32_t ow = (pt % a.ow_tiles) * a.box_w + r_w;
        pt /= a.ow_tiles;
        const uint32_t oh = (pt % a.oh_tiles) * a.rows + r_h;
        const uint32_t img = (pt / a.oh_tiles) * a.box_n + r_n;
        valid[mt] = tile_ok && rr < loaded_rows && r_w < a.box_w && ow < a.w_out && oh < a.h_out && img < a.n_img;
        obase[mt] = valid[mt] ? static_cast<int64_t>(img) * a.co * a.hw + static_cast<int64_t>(oh) * a.w_out + ow : 0;
      }
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * (MT * kAccN);
      if constexpr (TN2) {
        // out[p] = D[p][co] + D[p+1][64 + co]: row p+1 is the next lane, or for lane 31 the first
        // row of the next quarter, passed through smem (row 127 is never an output: qmax >= 1)
        const int half = (warp - 4) / 4;
        float* xb = xch + acc * (MT * 2 * 4 * 32);  // [mt][half][quarter][32 columns]
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int jj = 0; jj < N / 2; jj += 16) {
            uint32_t e[16];
            tmem_ld16(taddr + mt * kAccN + N + j_lo + jj, e);
            if (lane == 0) {
#pragma unroll
              for (int q = 0; q < 16; ++q) xb[((mt * 2 + half) * 4 + quarter) * 32 + jj + q] = __uint_as_float(e[q]);
            }
          }
        asm volatile("bar.sync 1, %0;\n" ::"r"(kEpiWarps * 32) : "memory");
#pragma unroll
        for (int jj = 0; jj < N / 2; jj += 16) {
          const int j0 = j_lo + jj;
          const uint32_t m0 = co_blk * N + j0;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            uint32_t d[16], e[16];
            tmem_ld16(taddr + mt * kAccN + j0, d);
            tmem_ld16(taddr + mt * kAccN + N + j0, e);
            const float* nx = xb + ((mt * 2 + half) * 4 + (quarter + 1 < 4 ? quarter + 1 : quarter)) * 32 + jj;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              float en = __shfl_down_sync(0xffffffffu, __uint_as_float(e[q]), 1);
              if (lane == 31) en = nx[q];
              if (valid[mt] && m0 + q < a.co)
                st_out(a.out + obase[mt] + static_cast<int64_t>(m0 + q) * a.hw, __uint_as_float(d[q]) + en);
            }
          }
        }
      } else
#pragma unroll
      for (int jj = 0; jj < N / 2; jj += 16) {
        const int j0 = j_lo + jj;
        uint32_t v[MT][16];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) tmem_ld16(taddr + mt * N + j0, v[mt]);
        const uint32_t m0 = co_blk * N + j0;
#ifndef IM2WIN_PHASE_NOSTORE  // exploration builds only: times the kernel without its output stores
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          if (m0 + q < a.co) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
              if (valid[mt]) st_out(a.out + obase[mt] + static_cast<int64_t>(m0 + q) * a.hw, __uint_as_float(v[mt][q]));
          }
        }
#else
        if (valid[0] && v[0][0] == 0x7fffffffu) a.out[obase[0]] = 0.f;
#endif
      }
#else
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        uint32_t pt = (PAIR ? pair * 2 + rank : pair) * MT + mt;
        const bool tile_ok = pt < a.p_tiles;
        const uint32_t ow = (pt % a.ow_tiles) * a.box_w + r_w;
        pt /= a.ow_tiles;
        const uint32_t oh = (pt % a.oh_tiles) * a.rows + r_h;
        const uint32_t img = (pt / a.oh_tiles) * a.box_n + r_n;
        const bool valid =
            tile_ok && rr < loaded_rows && r_w < a.box_w && ow < a.w_out && oh < a.h_out && img < a.n_img;
        const int64_t obase =
            valid ? static_cast<int64_t>(img) * a.co * a.hw + static_cast<int64_t>(oh) * a.w_out + ow : 0;
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * (MT * N) + mt * N;
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
      }
#endif
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR && rank != 0) mbar_arrive_remote(mapa_shared(&tempty_bar[acc], 0));
        else mbar_arrive(&tempty_bar[acc]);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // no CTA frees TMEM or exits while its peer may still signal it
  if (warp == 2) {
    tc_fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

// Pixel tile for the phase kernel; returns the fraction of the 128 MMA rows that are real outputs.
inline double phase_tile(int64_t n, int64_t h_out, int64_t w_out, int64_t qmax, PhaseArgs& a) {
  const int64_t max_w = kTileM - qmax;
  if (w_out <= max_w) {
    a.box_w = static_cast<uint32_t>(w_out);
    a.pitch = static_cast<uint32_t>(w_out + qmax);
    const int64_t rmax = std::max<int64_t>(1, kTileM / a.pitch);
    a.rows = static_cast<uint32_t>(std::min<int64_t>(h_out, rmax));
    a.box_n = a.rows == h_out
                  ? static_cast<uint32_t>(std::max<int64_t>(1, std::min<int64_t>(n, kTileM / (a.pitch * h_out))))
                  : 1u;
  } else {
    const int64_t parts = (w_out + max_w - 1) / max_w;
    a.box_w = static_cast<uint32_t>((w_out + parts - 1) / parts);
    a.pitch = static_cast<uint32_t>(a.box_w + qmax);
    a.rows = 1;
    a.box_n = 1;
  }
  return static_cast<double>(a.box_w) * a.rows * a.box_n / kTileM;
}

template <bool BF16, int N, int STAGES, int TAPS, int MT, bool PAIR = false, bool TN2 = false>
static int launch_phase(PhaseArgs a, const void* x_cl, const void* packed, int64_t c_pad, int64_t h, int64_t w,
                        int64_t Mp, int64_t Kp, const NhwcFeed& feed, cudaStream_t stream, const char** err) {
  constexpr int kBK = BF16 ? 64 : 32;
  auto enc = get_encode_fn();
  if (!enc) {
    *err = "conv_tc_phase: cuTensorMapEncodeTiled unavailable";
    return 2;
  }
  const cuuint64_t esz = BF16 ? 2 : 4;
  const CUtensorMapDataType dt = BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const int64_t s = a.stride;
  CUtensorMap map_a[2], map_b;
  for (int r = 0; r < 2; ++r) {
    const int rr = r < s ? r : 0;  // unused second map for stride 1
    cuuint64_t dims[5] = {static_cast<cuuint64_t>(c_pad), static_cast<cuuint64_t>((w - rr + s - 1) / s),
                          static_cast<cuuint64_t>(s), static_cast<cuuint64_t>((h + s - 1) / s), a.n_img};
    cuuint64_t strides[4] = {static_cast<cuuint64_t>(s * c_pad) * esz, static_cast<cuuint64_t>(w * c_pad) * esz,
                             static_cast<cuuint64_t>(s * w * c_pad) * esz, static_cast<cuuint64_t>(h * w * c_pad) * esz};
    cuuint32_t box[5] = {static_cast<cuuint32_t>(kBK), a.pitch, 1, a.rows, a.box_n};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    const char* base = static_cast<const char*>(x_cl) + rr * c_pad * esz;
    CUresult res = enc(&map_a[r], dt, 5, const_cast<char*>(base), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS) {
      *err = "conv_tc_phase: input tensor map rejected (cuTensorMapEncodeTiled)";
      return 2;
    }
  }
  {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(Mp)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(Kp) * esz};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(PAIR && !TN2 ? N / 2 : N)};
    cuuint32_t estr[2] = {1, 1};
    CUresult res = enc(&map_b, dt, 2, const_cast<void*>(packed), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS) {
      *err = "conv_tc_phase: filter tensor map rejected (cuTensorMapEncodeTiled)";
      return 2;
    }
  }
  a.co_tiles = static_cast<uint32_t>(Mp / N);
  const int b_rows = PAIR && TN2 ? (TAPS + 1) / 2 * N : TAPS * (PAIR ? N / 2 : N);  // staged filter rows
  const size_t smem = static_cast<size_t>(STAGES) * (MT * kPhRows + b_rows) * kRowBytes + 1024;
  a.k_total = static_cast<uint32_t>(Kp);
  auto kern = conv_tc_phase_kernel<BF16, N, STAGES, TAPS, MT, PAIR, TN2>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 2;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t items = static_cast<uint64_t>(a.pairs) * a.co_tiles;
  uint32_t grid = items < static_cast<uint64_t>(sms) ? static_cast<uint32_t>(items) : static_cast<uint32_t>(sms);
  if constexpr (PAIR) {
    const int clusters = max_pair_clusters(kern, smem, feed.src != nullptr);
    if (clusters < 1) {
      *err = "conv_tc_phase: no 2-CTA cluster fits";
      return 2;
    }
    grid = 2 * static_cast<uint32_t>(std::min<uint64_t>(items, static_cast<uint64_t>(clusters)));
    im2win_note_kernel(TN2 ? "conv_tc_phase_kernel (phase shift, CTA pair M=256 x tap pairs N=128, 2 tiles/CTA)"
                       : MT == 4 ? "conv_tc_phase_kernel (phase shift, CTA pair M=256, 4 tiles/CTA)"
                                 : "conv_tc_phase_kernel (phase shift, CTA pair M=256, 2 tiles/CTA)");
  } else if (TN2) {
    im2win_note_kernel("conv_tc_phase_kernel (phase shift, tap pairs N=128, 2 tiles/item)");
  } else {
    im2win_note_kernel(MT == 4 ? "conv_tc_phase_kernel (phase shift, 4 tiles/item)"
                               : "conv_tc_phase_kernel (phase shift, 2 tiles/item)");
  }
  e = launch_tc_kernel(kern, grid, smem, stream, feed.src != nullptr, PAIR ? 2 : 1, a, map_a[0], map_a[1], map_b,
                       feed_for(feed, PAIR ? grid / 2 : grid, items));
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

// B[m][(fh*Wf + fw)*Kc + c] = F[m][c][fh][fw] (zero for c >= C) -- same packing as the shift kernel.
template <bool BF16>
__global__ void pack_filter_phase_kernel(const float* __restrict__ flt, void* __restrict__ packed, int M, int C,
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

}  // namespace tc
}  // namespace im2win

// Returns 1 and launches when the phase kernel applies, 0 when the caller should try the
// next kernel, <0 on error.  Applies to stride 1-2, Wf in {3, 5, 7}, channel pitch >= 32
// (a K-slab is one channel chunk of one tap), Co <= 128.
int im2win_try_conv_tc_phase(const void* x_cl, const float* flt, float* out, void* workspace, int64_t n, int64_t c_in,
                             int64_t c_pad, int64_t h, int64_t w, int64_t c_out, int h_f, int w_f, int stride, int bf16,
                             double fused_util, const im2win::tc::NhwcFeed& feed, cudaStream_t stream,
                             const char** err) {
  using namespace im2win::tc;
  const char* env = getenv("IM2WIN_PHASE");
  const int mode = env ? atoi(env) : 1;  // 0: off, 1: auto, 2: force where legal (tests)
  if (mode == 0) return 0;
  // measured (tools/tc_kernels.py, N=128): stride 2 (conv4, Co=64) 1.57x over the generic fused
  // kernel; stride 1 with Co=64 (conv9, 4 tiles per item) 1.09x over the window-shift kernel;
  // stride 1 with Co=128: the shift kernel (conv_tc_shift.cu) is faster for BF16 (conv8 868 vs 829
  // TF) and for small outputs (conv10); TF32 on wide outputs prefers the phase kernel (conv8 528 vs 493)
  if (mode == 1 && stride == 1 && c_out > 64 && (bf16 || (w - w_f + 1) < 64)) return 0;
  if (stride < 1 || stride > 2 || (w_f != 3 && w_f != 5 && w_f != 7) || c_out > 128) return 0;
  const int bk = bf16 ? 64 : 32;
  if (c_pad < 32) return 0;
  const int64_t h_out = (h - h_f) / stride + 1, w_out = (w - w_f) / stride + 1;
  const int64_t qmax = (w_f - 1) / stride;
  const int taps = (w_f + stride - 1) / stride;
  PhaseArgs a{};
  a.out = out;
  a.n_img = static_cast<uint32_t>(n);
  a.h_out = static_cast<uint32_t>(h_out);
  a.w_out = static_cast<uint32_t>(w_out);
  a.hw = static_cast<uint32_t>(h_out * w_out);
  a.co = static_cast<uint32_t>(c_out);
  const double util = phase_tile(n, h_out, w_out, qmax, a);
  if (mode == 1 && util + 1e-9 < fused_util * 0.9) return 0;
  const int N = c_out <= 64 ? 64 : 128;
  if (N == 128 && taps >= 5) return 0;  // a stage would not fit twice in shared memory
  // boxes of several output rows may overhang the last row; with h % s != 0 the phase view
  // could then address one row past the tensor -- keep to whole-row tiles there
  if (h % stride != 0 && a.rows > 1 && h_out % a.rows != 0) return 0;
  const int64_t c_slabs = (c_pad + bk - 1) / bk;
  const int64_t Kc = c_slabs * bk;
  const int64_t Kp = static_cast<int64_t>(h_f) * w_f * Kc;
  const int64_t Mp = (c_out + N - 1) / N * N;
  a.ow_tiles = (a.w_out + a.box_w - 1) / a.box_w;
  a.oh_tiles = (a.h_out + a.rows - 1) / a.rows;
  a.n_tiles = (a.n_img + a.box_n - 1) / a.box_n;
  a.p_tiles = a.ow_tiles * a.oh_tiles * a.n_tiles;
  // pixel tiles per work item: every staged filter tile feeds mt MMAs.  Measured on conv4 BF16
  // (N=128): 1 -> 570, 2 -> 724, 4 -> 835 TF; 4 tiles x 2 x 64 fp32 columns fill TMEM exactly.
  const char* mt_env = getenv("IM2WIN_PHASE_MT");
  int mt_sel = (N == 64 && taps <= 5) ? 4 : 2;
  if (mt_env && (atoi(mt_env) == 2 || (atoi(mt_env) == 4 && N == 64 && taps <= 5))) mt_sel = atoi(mt_env);
  // CTA pairs (cta_group::2, M = 256): IM2WIN_PAIR=1 turns them on; off by default.  Measured
  // (tools/probes/umma_rate.cu, B200): a 128x64x16 BF16 UMMA from shared memory takes 48 cycles
  // (operand-read bound: 6 KB at 128 B/clk; 32 cycles of math), the pair's 256x64x16 44.6 --
  // the B half the pair saves is not what bounds it, and conv4/conv9 time the same with and
  // without pairs (BF16 conv4 0.819 vs 0.811 ms, N=128); conv8 TF32 (N=128) 2% faster.
  const char* pair_env = getenv("IM2WIN_PAIR");
  const bool pair = pair_env && atoi(pair_env) > 0;
  // tap pairs per MMA for Co <= 64 (2 pixel tiles per item).  Measured (tools/tn2_ab.py, conv
  // alone): 4 taps per phase (conv4, 7x7 stride 2) BF16 817 -> 944 TF at N=128, 862 -> 953 at 512,
  // 874 -> 881 at 2048; TF32 +11-26%; 3 taps (conv9, 3x3 stride 1) TF32 +3-6% but BF16 -8% (fewer
  // taps to pair, half the filter reuse of 4 tiles per item).  IM2WIN_PHASE_TN2: 0 off, 1 auto, 2
  // wherever legal.
  const char* tn2_env = getenv("IM2WIN_PHASE_TN2");
  const int tn2_mode = tn2_env ? atoi(tn2_env) : 1;
  const bool tn2 = N == 64 && taps >= 2 && taps <= 4 &&
                   (tn2_mode == 2 || (tn2_mode == 1 && (taps == 4 || (!bf16 && taps == 3))));
  if (tn2) mt_sel = 2;
  a.pairs = (a.p_tiles + mt_sel * (pair ? 2 : 1) - 1) / (mt_sel * (pair ? 2 : 1));
  a.stride = static_cast<uint32_t>(stride);
  a.w_f = static_cast<uint32_t>(w_f);
  a.c_slabs = static_cast<uint32_t>(c_slabs);
  a.k_iters = static_cast<uint32_t>(h_f * stride * c_slabs);
  if (bf16)
    pack_filter_phase_kernel<true><<<256, 256, 0, stream>>>(flt, workspace, static_cast<int>(c_out),
                                                            static_cast<int>(c_in), h_f, w_f, static_cast<int>(Mp),
                                                            static_cast<int>(Kc));
  else
    pack_filter_phase_kernel<false><<<256, 256, 0, stream>>>(flt, workspace, static_cast<int>(c_out),
                                                             static_cast<int>(c_in), h_f, w_f, static_cast<int>(Mp),
                                                             static_cast<int>(Kc));
  int rc = 1;
  if (tn2) {
    // stage = 2 x 17 KB of A + taps x 8 KB of B (+ 4 KB static exchange buffer)
#define IM2WIN_PHT(BF, ST, TP)                                                                               \
  rc = pair ? launch_phase<BF, 64, 4, TP, 2, true, true>(a, x_cl, workspace, c_pad, h, w, Mp, Kp, feed, stream, err) \
            : launch_phase<BF, 64, ST, TP, 2, false, true>(a, x_cl, workspace, c_pad, h, w, Mp, Kp, feed, stream, err)
    if (bf16) {
      if (taps == 2) IM2WIN_PHT(true, 4, 2);
      else if (taps == 3) IM2WIN_PHT(true, 3, 3);
      else IM2WIN_PHT(true, 3, 4);
    } else {
      if (taps == 2) IM2WIN_PHT(false, 4, 2);
      else if (taps == 3) IM2WIN_PHT(false, 3, 3);
      else IM2WIN_PHT(false, 3, 4);
    }
#undef IM2WIN_PHT
    return rc == 0 ? 1 : -rc;
  }
  // stage = 2 x 17 KB of A + taps x N x 128 B of B; as many stages as fit in 227 KB
#define IM2WIN_PH(BF, NN, ST, TP)                                                                             \
  rc = pair ? launch_phase<BF, NN, ST, TP, 2, true>(a, x_cl, workspace, c_pad, h, w, Mp, Kp, feed, stream, err) \
            : launch_phase<BF, NN, ST, TP, 2>(a, x_cl, workspace, c_pad, h, w, Mp, Kp, feed, stream, err)
#define IM2WIN_PH_T(BF)                                        \
  switch (taps * 1000 + N) {                                   \
    case 2064: IM2WIN_PH(BF, 64, 4, 2); break;                 \
    case 2128: IM2WIN_PH(BF, 128, 3, 2); break;                \
    case 3064: IM2WIN_PH(BF, 64, 3, 3); break;                 \
    case 3128: IM2WIN_PH(BF, 128, 2, 3); break;                \
    case 4064: IM2WIN_PH(BF, 64, 3, 4); break;                 \
    case 4128: IM2WIN_PH(BF, 128, 2, 4); break;                \
    case 5064: IM2WIN_PH(BF, 64, 3, 5); break;                 \
    case 7064: IM2WIN_PH(BF, 64, 2, 7); break;                 \
    default: break;                                            \
  }
  if (mt_sel == 4) {
    // stage = 4 x 17 KB of A + taps x 8 KB of B: two stages
#define IM2WIN_PH4_T(BF, TP)                                                                                \
  rc = pair ? launch_phase<BF, 64, 2, TP, 4, true>(a, x_cl, workspace, c_pad, h, w, Mp, Kp, feed, stream, err) \
            : launch_phase<BF, 64, 2, TP, 4>(a, x_cl, workspace, c_pad, h, w, Mp, Kp, feed, stream, err)
#define IM2WIN_PH4(BF)                          \
  switch (taps) {                               \
    case 2: IM2WIN_PH4_T(BF, 2); break;         \
    case 3: IM2WIN_PH4_T(BF, 3); break;         \
    case 4: IM2WIN_PH4_T(BF, 4); break;         \
    default: IM2WIN_PH4_T(BF, 5); break;        \
  }
    if (bf16) {
      IM2WIN_PH4(true)
    } else {
      IM2WIN_PH4(false)
    }
#undef IM2WIN_PH4
#undef IM2WIN_PH4_T
  } else if (bf16) {
    IM2WIN_PH_T(true)
  } else {
    IM2WIN_PH_T(false)
  }
#undef IM2WIN_PH_T
#undef IM2WIN_PH
  return rc == 0 ? 1 : -rc;
}
