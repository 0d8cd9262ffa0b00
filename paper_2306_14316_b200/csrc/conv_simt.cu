// FP32 CUDA-core im2win convolution (paper Alg. 3) for sm_100a.
//
// Restates winconv `_tiled_kernel` (reference pkg/src/winconv/kernels/optimized.py:66-214):
// the GEMM  O[m, n] = sum_k F[m, k] * W[k, n]  with M = Co, N = batch*Ho*Wo,
// K = Ci*Hf*Wf (kernels/reference.py:30-46), where the logical window matrix
// W[k, n] = I~[src_off(n) + delta(k)] is read straight out of the im2win tensor
// (optimized.py:30-50, :93-106).
//
// Arithmetic contract (bit-exact with the reference): every output element is a
// float32 chain  acc = +0;  for k ascending: acc = acc + rn(F*W)  with an
// UNFUSED multiply and add (reference optimized.py:162-165, reference.py:4-8).
// EXACT=true emits FMUL+FADD (__fmul_rn/__fadd_rn are never contracted);
// EXACT=false is the optional FFMA variant (within 1e-4, not bit-exact).
// There is no split-K: one thread owns each output element for the whole K loop.
//
// Blackwell structure (paper Alg. 3 re-done):
//   * CTA tile BM x BN, K-slab BK, STAGES-deep cp.async ring in shared memory
//     (the "prefetch / double buffer" of the paper; STAGES=1 disables it);
//   * the filter is pre-packed once per call into a zero-padded K-major panel
//     FT[Kp][Mp] so its slabs are 16-byte async copies;
//   * the window panel is gathered 4 bytes at a time with zero fill, using a
//     per-k offset table delta[k] and per-column base pointers src_off(n)
//     (the reference's hoisted src_off/delta, optimized.py:42, :101-102);
//   * register micro-kernel: each thread owns an 8x8 tile split into two 4x4
//     quadrants so fragments are 128-bit shared loads ("vectorized load").
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

#ifndef IM2WIN_SIMT_BRANCHLESS
#define IM2WIN_SIMT_BRANCHLESS 1  // measured +0.7% on the 12-layer step (fewer branch/convergence ops)
#endif
#ifndef IM2WIN_SIMT_NOCLAMP
#define IM2WIN_SIMT_NOCLAMP 0  // padded k: ignore-src predicate only, no address clamp
#endif
#ifndef IM2WIN_SIMT_PART_ROWS
#define IM2WIN_SIMT_PART_ROWS 4  // window rows gathered per interleaved hook
#endif
#ifndef IM2WIN_SIMT_SMALLK
#define IM2WIN_SIMT_SMALLK 1  // persistent small-K kernel for K <= 64, Co <= 64 (conv7)
#endif
#ifndef IM2WIN_SIMT_SMALLK_UNROLL
#define IM2WIN_SIMT_SMALLK_UNROLL 4
#endif
#ifndef IM2WIN_SIMT_MINB192
#define IM2WIN_SIMT_MINB192 2  // resident CTAs asked of the 192-thread 96x128 tile (register cap)
#endif
#ifndef IM2WIN_SIMT_INTERLEAVE
#define IM2WIN_SIMT_INTERLEAVE 1
#endif
#ifndef IM2WIN_SIMT_KTAIL
#define IM2WIN_SIMT_KTAIL 1  // padded last K slab computed over its real rows only
#endif
#ifndef IM2WIN_SIMT_SDELTA
#define IM2WIN_SIMT_SDELTA 1
#endif

namespace im2win {

struct ConvArgs {
  const float* __restrict__ win;    // im2win tensor, flat
  const float* __restrict__ fltT;   // packed filter [Kp][Mp]
  const int* __restrict__ delta;    // [Kp], -1 beyond K
  float* __restrict__ out;          // (N, Co, Ho, Wo)
  int M, Mp, K, Kp;
  uint32_t n_gemm;                  // N*Ho*Wo
  uint32_t c_in, h_out, w_out, row_len, s_hf, hw;
  // GEMM column n = (img, oh, ow) starts at img*img_stride + oh*row_stride + ow*col_stride in the
  // source: the im2win tensor Ĩ (c_in*h_out*row_len, row_len, s*Hf) or, for the no-Ĩ entry point,
  // the NCHW input itself (C*H*W, s*W, s) -- the same window elements, so the same bits
  uint32_t img_stride, row_stride, col_stride;
  FastDiv fd_hw, fd_wo;
  uint32_t m_tiles;
  uint32_t vec_out;                 // Ho*Wo % 4 == 0: 16-byte output stores
  uint32_t n_base;                  // first GEMM column of this launch (tail launches)
  uint32_t m_base;                  // first output channel of this launch (row-split launches)
  uint32_t co_out;                  // output channels (image stride / hw); M may stop short of it
  float neg_zero, one;              // -0.0f and 1.0f, opaque to the compiler (packed exact MACs)
};

// ---------------------------------------------------------------------------
// pack: FT[k][m] = F[m][k] (zero padded), delta[k] = c*chan_stride + fh*fh_stride + fw*fw_stride
// (Ĩ: c*Ho*RL + fw*Hf + fh; NCHW input: c*H*W + fh*W + fw)
// ---------------------------------------------------------------------------
__global__ void pack_filter_kernel(const float* __restrict__ flt, float* __restrict__ fltT,
                                   int* __restrict__ delta, int M, int K, int Mp, int Kp, int h_f,
                                   int w_f, int chan_stride, int fh_stride, int fw_stride) {
  const int64_t total = static_cast<int64_t>(Kp) * Mp;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int k = static_cast<int>(i / Mp);
    int m = static_cast<int>(i % Mp);
    fltT[i] = (k < K && m < M) ? flt[static_cast<int64_t>(m) * K + k] : 0.0f;
    if (m == 0) {
      int d = -1;
      if (k < K) {
        int fhw = h_f * w_f;
        int c = k / fhw, r = k % fhw;
        int fh = r / w_f, fw = r % w_f;
        d = c * chan_stride + fh * fh_stride + fw * fw_stride;
      }
      delta[k] = d;
    }
  }
}

template <bool EXACT>
IM2WIN_DEVICE float mac(float acc, float a, float b) {
  if constexpr (EXACT) {
    return __fadd_rn(acc, __fmul_rn(a, b));
  } else {
    return __fmaf_rn(a, b, acc);
  }
}

#ifndef IM2WIN_SIMT_FP2
#define IM2WIN_SIMT_FP2 1  // exact multiply-then-add as two packed FFMA2 (0: scalar FMUL + FADD)
#endif

// One micro-tile row: acc[j] = rn(acc[j] + rn(a * fb[j])), ascending k per element (the caller's
// k loop).  IM2WIN_SIMT_FP2: the same two roundings per element through the packed sm_100
// FMUL2/FADD2 (per component identical to __fmul_rn/__fadd_rn): half the FP instructions.
template <bool EXACT, int MT, bool FP2 = IM2WIN_SIMT_FP2>
IM2WIN_DEVICE void mac_row(float (&acc)[MT], float a, const float (&fb)[MT], float nz, float one) {
#if IM2WIN_SIMT_FP2
  if constexpr (EXACT && FP2) {
    // rn(a*b) = fma(a, b, -0) and rn(c + p) = fma(c, 1, p) exactly (signed zeros included); -0
    // and 1 arrive as kernel arguments so ptxas cannot see through them and contract the pair
    // into one FFMA2 (it fuses mul.rn.f32x2 + add.rn.f32x2 and the __fmul2_rn/__fadd2_rn pair)
#pragma unroll
    for (int j = 0; j < MT; j += 2) {
      uint64_t p, c;
      asm("{\n\t.reg .b64 aa, bb, zz;\n\tmov.b64 aa, {%1, %1};\n\tmov.b64 bb, {%2, %3};\n\t"
          "mov.b64 zz, {%4, %4};\n\tfma.rn.f32x2 %0, aa, bb, zz;\n\t}\n"
          : "=l"(p) : "f"(a), "f"(fb[j]), "f"(fb[j + 1]), "f"(nz));
      asm("{\n\t.reg .b64 cc, oo;\n\tmov.b64 cc, {%1, %2};\n\tmov.b64 oo, {%4, %4};\n\t"
          "fma.rn.f32x2 %0, cc, oo, %3;\n\t}\n"
          : "=l"(c) : "f"(acc[j]), "f"(acc[j + 1]), "l"(p), "f"(one));
      asm("mov.b64 {%0, %1}, %2;\n" : "=f"(acc[j]), "=f"(acc[j + 1]) : "l"(c));
    }
    return;
  }
  if constexpr (!EXACT && FP2) {
    // the FFMA variant: one packed FFMA2 per pair (per component the same as __fmaf_rn)
#pragma unroll
    for (int j = 0; j < MT; j += 2) {
      uint64_t c;
      asm("{\n\t.reg .b64 aa, bb, cc;\n\tmov.b64 aa, {%1, %1};\n\tmov.b64 bb, {%2, %3};\n\t"
          "mov.b64 cc, {%4, %5};\n\tfma.rn.f32x2 %0, aa, bb, cc;\n\t}\n"
          : "=l"(c) : "f"(a), "f"(fb[j]), "f"(fb[j + 1]), "f"(acc[j]), "f"(acc[j + 1]));
      asm("mov.b64 {%0, %1}, %2;\n" : "=f"(acc[j]), "=f"(acc[j + 1]) : "l"(c));
    }
    return;
  }
#endif
  (void)nz;
  (void)one;
#pragma unroll
  for (int j = 0; j < MT; ++j) acc[j] = mac<EXACT>(acc[j], a, fb[j]);
}

// MT: register micro-tile MT x MT per thread (8: two 4x4 quadrants, the paper's
// 8x8; 4: one 4x4 quadrant, for layers too small to fill 148 SMs with 8x8 threads).
// SD: the per-k offset table delta[] is staged in shared memory once per CTA
// (its global-load latency otherwise sits on the gather's critical path).
// The gather of slab kt+STAGES-1 is issued in BK/4 parts interleaved with the
// compute of slab kt, so the 4-byte async copies do not arrive as one burst.
// PADK: K is not a multiple of BK, so the last slab holds padded k (delta -1, zero fill).
// Without padded k every gathered element is a plain copy: no per-element predicate.
template <int BM, int BN, int BK, int STAGES, bool EXACT, bool VEC, int MT, bool SD, bool PADK = true>
__global__ void __launch_bounds__((BM / MT) * (BN / MT), MT == 8 ? ((BM / MT) * (BN / MT) <= 192 ? IM2WIN_SIMT_MINB192 : 2) : ((BM / MT) * (BN / MT) >= 512 ? 1 : 3))
    conv_simt_kernel(const ConvArgs a) {
  constexpr int NT = (BM / MT) * (BN / MT);
  constexpr int TXN = BN / MT;                // threads along n
  constexpr int CPT = (BN + NT - 1) / NT;     // gather columns per thread
  constexpr int HALVES = MT / 4;              // 4-wide quadrants per axis
  constexpr int PR = IM2WIN_SIMT_PART_ROWS;   // window rows per gather part
  constexpr int PARTS = BK / PR;              // gather parts per slab
  // packed exact MACs everywhere but the 96-row tile (conv1/conv2: 3-5% slower with them)
  constexpr bool kFP2 = IM2WIN_SIMT_FP2 && BM != 96;
  static_assert(PR % 4 == 0 && BK % PR == 0, "parts are whole int4 delta loads");
  static_assert(MT == 4 || MT == 8, "micro-tile is 4x4 or 8x8");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* As = reinterpret_cast<float*>(smem_raw);  // [STAGES][BK][BM]
  float* Bs = As + STAGES * BK * BM;               // [STAGES][BK][BN]
  int* sdelta = reinterpret_cast<int*>(Bs + STAGES * BK * BN);  // [Kp] when SD

  const int tid = threadIdx.x;
  const uint32_t m_tile = blockIdx.x % a.m_tiles;
  const uint32_t n_tile = blockIdx.x / a.m_tiles;
  const int m0 = a.m_base + m_tile * BM;
  const uint32_t n0 = a.n_base + n_tile * BN;

  if constexpr (SD) {
    for (int q = tid; q < a.Kp / 4; q += NT)
      reinterpret_cast<int4*>(sdelta)[q] = __ldg(reinterpret_cast<const int4*>(a.delta) + q);
    __syncthreads();
  }
  const int* dtab = SD ? sdelta : a.delta;

  // Per-thread gather columns: the window-matrix column n starts at
  // src_off(n) = ((img*C*Ho + oh)*RL + ow*s*Hf) (optimized.py:101-102);
  // element (k, n) is src_off(n) + delta[k].  Columns past N zero-fill.
  const float* bsrc[CPT];
  bool bzero[CPT];
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    const uint32_t n = n0 + tid + j * NT;
    bsrc[j] = a.win;
    bzero[j] = true;
    if (tid + j * NT < BN && n < a.n_gemm) {
      uint32_t img, rem, oh, ow;
      a.fd_hw.divmod(n, img, rem);
      a.fd_wo.divmod(rem, oh, ow);
      bsrc[j] = a.win + static_cast<int64_t>(img) * a.img_stride + static_cast<int64_t>(oh) * a.row_stride +
                static_cast<int64_t>(ow) * a.col_stride;
      bzero[j] = false;
    }
  }

  const int k_tiles = a.Kp / BK;
  const int k_full = a.K / BK;  // slabs with no padded k

  // filter slab: BK rows of BM floats, 16-byte copies
  auto load_filter = [&](int kt, int slot) {
    const float* fsrc = a.fltT + static_cast<int64_t>(kt) * BK * a.Mp + m0;
    float* adst = As + slot * BK * BM;
#pragma unroll
    for (int q = tid; q < BK * BM / 4; q += NT) {
      int r = q / (BM / 4), c4 = q % (BM / 4);
      cp_async_16(smem_u32(adst + r * BM + c4 * 4), fsrc + static_cast<int64_t>(r) * a.Mp + c4 * 4, 16);
    }
  };
  // window slab rows [4*part, 4*part+4): each gathering thread owns whole columns
  auto load_window_part = [&](int kt, int slot, int part) {
    int d[PR];
#pragma unroll
    for (int q = 0; q < PR / 4; ++q) {
      const int4 v = SD ? *reinterpret_cast<const int4*>(dtab + kt * BK + PR * part + 4 * q)
                        : __ldg(reinterpret_cast<const int4*>(dtab + kt * BK + PR * part + 4 * q));
      d[4 * q] = v.x; d[4 * q + 1] = v.y; d[4 * q + 2] = v.z; d[4 * q + 3] = v.w;
    }
    float* bdst = Bs + slot * BK * BN + PR * part * BN;
    const bool full = kt < k_full;
#if IM2WIN_SIMT_BRANCHLESS
    // branch-free form: every element predicated (padded k -> delta -1 -> zero fill)
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int c = tid + j * NT;
      if (CPT * NT == BN || c < BN) {
#pragma unroll
        for (int kk = 0; kk < PR; ++kk) {
          if constexpr (!PADK) {
            // columns past N (bzero) read image 0's window: valid memory, never stored
            cp_async_4_zfill(smem_u32(bdst + kk * BN + c), bsrc[j] + d[kk], bzero[j]);
            continue;
          }
          const bool ok = d[kk] >= 0;
#if IM2WIN_SIMT_NOCLAMP
          // ignore-src copies never touch the source: the address need not be valid
          cp_async_4_zfill(smem_u32(bdst + kk * BN + c), bsrc[j] + d[kk], bzero[j] || !ok);
#else
          cp_async_4_zfill(smem_u32(bdst + kk * BN + c), bsrc[j] + (ok ? d[kk] : 0), bzero[j] || !ok);
#endif
        }
      }
    }
    (void)full;
#else
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int c = tid + j * NT;
      if (c < BN) {
        if (full) {
#pragma unroll
          for (int kk = 0; kk < PR; ++kk) cp_async_4_zfill(smem_u32(bdst + kk * BN + c), bsrc[j] + d[kk], bzero[j]);
        } else {
#pragma unroll
          for (int kk = 0; kk < PR; ++kk) {
            const bool ok = d[kk] >= 0;
            cp_async_4_zfill(smem_u32(bdst + kk * BN + c), ok ? bsrc[j] + d[kk] : a.win, bzero[j] || !ok);
          }
        }
      }
    }
#endif
  };
  auto load_stage = [&](int kt, int slot) {
    load_filter(kt, slot);
#pragma unroll
    for (int p = 0; p < PARTS; ++p) load_window_part(kt, slot, p);
  };

  float acc[MT][MT];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < MT; ++j) acc[i][j] = 0.0f;

  const int tx = tid % TXN;
  const int ty = tid / TXN;

  // compute one slab; `hook(p)` runs before k-step 4p (issues prefetch part p)
  auto compute_stage = [&](int slot, auto&& hook) {
    const float* as = As + slot * BK * BM;
    const float* bs = Bs + slot * BK * BN;
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      if (kk % PR == 0) hook(kk / PR);
      float fa[MT], fb[MT];
      if constexpr (VEC) {
#pragma unroll
        for (int h = 0; h < HALVES; ++h) {
          float4 av = *reinterpret_cast<const float4*>(as + kk * BM + h * (BM / 2) + ty * 4);
          float4 bv = *reinterpret_cast<const float4*>(bs + kk * BN + h * (BN / 2) + tx * 4);
          fa[4 * h] = av.x; fa[4 * h + 1] = av.y; fa[4 * h + 2] = av.z; fa[4 * h + 3] = av.w;
          fb[4 * h] = bv.x; fb[4 * h + 1] = bv.y; fb[4 * h + 2] = bv.z; fb[4 * h + 3] = bv.w;
        }
      } else {
#pragma unroll
        for (int h = 0; h < HALVES; ++h)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            fa[4 * h + i] = as[kk * BM + h * (BM / 2) + ty * 4 + i];
            fb[4 * h + i] = bs[kk * BN + h * (BN / 2) + tx * 4 + i];
          }
      }
#pragma unroll
      for (int i = 0; i < MT; ++i) mac_row<EXACT, MT, kFP2>(acc[i], fa[i], fb, a.neg_zero, a.one);
    }
  };
  auto no_hook = [](int) {};

  if constexpr (STAGES == 1) {
    for (int kt = 0; kt < k_tiles; ++kt) {
      load_stage(kt, 0);
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      compute_stage(0, no_hook);
      __syncthreads();
    }
  } else {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < k_tiles) load_stage(s, s);
      cp_async_commit();
    }
    int slot = 0, pslot = STAGES - 1;
    // a last slab holding padded k runs after the loop over its real rows only (conv3: K = 147
    // in 10 slabs of 16 would be 8% padded multiply-adds)
    const bool k_tail = IM2WIN_SIMT_KTAIL && IM2WIN_SIMT_BRANCHLESS && VEC && PADK && a.K != a.Kp;
    const int k_main = k_tail ? k_tiles - 1 : k_tiles;
    for (int kt = 0; kt < k_main; ++kt) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      const int pf = kt + STAGES - 1;
      const bool do_pf = pf < k_tiles;
      // one copy of the unrolled compute body (a second, hook-less copy overflows the
      // instruction cache: measured as no_instructions stalls)
      if (do_pf) {
        if (IM2WIN_SIMT_INTERLEAVE) load_filter(pf, pslot);
        else load_stage(pf, pslot);
      }
#if IM2WIN_SIMT_BRANCHLESS
      // past the last slab the parts still run (uniform code, no branch in the unrolled body),
      // re-gathering the last slab into the slot that was just consumed -- never read again.
      // Measured: +0.7% on the step over the branched hook; a zero-fill flag instead costs more.
      const int pf_c = do_pf ? pf : k_tiles - 1;
      compute_stage(slot, [&](int p) { load_window_part(pf_c, pslot, p); });
#else
      compute_stage(slot, [&](int p) {
        if (IM2WIN_SIMT_INTERLEAVE && do_pf) load_window_part(pf, pslot, p);
      });
#endif
      cp_async_commit();
      slot = slot + 1 == STAGES ? 0 : slot + 1;
      pslot = pslot + 1 == STAGES ? 0 : pslot + 1;
    }
    if (k_tail) {
      // slab k_tiles-1 sits in `slot` (the loop's redundant re-gathers went to other slots);
      // skipping its zero rows changes no bits: acc never holds -0, so acc + rn(0*0) == acc
      cp_async_wait<0>();
      __syncthreads();
      const int krem = a.K - (k_tiles - 1) * BK;
      const float* as = As + slot * BK * BM;
      const float* bs = Bs + slot * BK * BN;
#pragma unroll 1
      for (int kk = 0; kk < krem; ++kk) {
        float fa[MT], fb[MT];
#pragma unroll
        for (int h = 0; h < HALVES; ++h) {
          float4 av = *reinterpret_cast<const float4*>(as + kk * BM + h * (BM / 2) + ty * 4);
          float4 bv = *reinterpret_cast<const float4*>(bs + kk * BN + h * (BN / 2) + tx * 4);
          fa[4 * h] = av.x; fa[4 * h + 1] = av.y; fa[4 * h + 2] = av.z; fa[4 * h + 3] = av.w;
          fb[4 * h] = bv.x; fb[4 * h + 1] = bv.y; fb[4 * h + 2] = bv.z; fb[4 * h + 3] = bv.w;
        }
#pragma unroll
        for (int i = 0; i < MT; ++i) mac_row<EXACT, MT, kFP2>(acc[i], fa[i], fb, a.neg_zero, a.one);
      }
    }
  }

#if IM2WIN_SIMT_BRANCHLESS
  cp_async_wait<0>();  // the redundant tail gathers must land before the CTA exits
#endif
  // epilogue: scatter to NCHW (optimized.py:209-214).  With Ho*Wo % 4 == 0 every
  // aligned group of 4 columns lies in one image and is 16-byte aligned: one
  // streaming 16-byte store per (row, quadrant).
#pragma unroll
  for (int hj = 0; hj < HALVES; ++hj) {
    const uint32_t nq = n0 + hj * (BN / 2) + tx * 4;  // first column of this quadrant
    if (a.vec_out && nq + 3 < a.n_gemm) {
      uint32_t img, rem;
      a.fd_hw.divmod(nq, img, rem);
      float* base = a.out + static_cast<int64_t>(img) * a.co_out * a.hw + rem;
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int m = m0 + (i / 4) * (BM / 2) + ty * 4 + (i % 4);
        if (m < a.M)
          __stcs(reinterpret_cast<float4*>(base + static_cast<int64_t>(m) * a.hw),
                 make_float4(acc[i][4 * hj], acc[i][4 * hj + 1], acc[i][4 * hj + 2], acc[i][4 * hj + 3]));
      }
    } else {
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const uint32_t n = nq + jj;
        if (n >= a.n_gemm) continue;
        uint32_t img, rem;
        a.fd_hw.divmod(n, img, rem);
        float* base = a.out + static_cast<int64_t>(img) * a.co_out * a.hw + rem;
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const int m = m0 + (i / 4) * (BM / 2) + ty * 4 + (i % 4);
          if (m < a.M) base[static_cast<int64_t>(m) * a.hw] = acc[i][4 * hj + jj];
        }
      }
    }
  }
}


// ---------------------------------------------------------------------------
// Small-K persistent variant (K <= 64, Co <= 64: conv7, K = 27).  With one or two
// K-slabs per tile the per-CTA prologue (first gathers) and epilogue (output stores)
// dominate a 64x256 CTA's life.  Here each CTA keeps its filter panel resident and
// walks n-tiles: the window gather of tile i+1 is in flight while tile i is computed
// and stored.  Same micro-tile, same arithmetic (FMUL+FADD in ascending k from +0),
// and the k loop stops at K instead of the padded Kp.
// ---------------------------------------------------------------------------
template <int KP, bool EXACT>
__global__ void __launch_bounds__(256, 2) conv_simt_smallk_kernel(const ConvArgs a) {
  constexpr int BM = 64, BN = 256, MT = 8, NT = 256, TXN = BN / MT;
  constexpr int kUnroll = IM2WIN_SIMT_SMALLK_UNROLL;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* As = reinterpret_cast<float*>(smem_raw);  // [KP][BM], resident
  float* Bs = As + KP * BM;                         // [2][KP][BN]
  int* sdelta = reinterpret_cast<int*>(Bs + 2 * KP * BN);  // [KP]
  const int tid = threadIdx.x;
  for (int q = tid; q < KP * BM / 4; q += NT)
    reinterpret_cast<float4*>(As)[q] = __ldg(reinterpret_cast<const float4*>(a.fltT) + q);  // Mp == BM
  for (int q = tid; q < KP; q += NT) sdelta[q] = __ldg(a.delta + q);
  __syncthreads();

  const uint32_t n_tiles = (a.n_gemm + BN - 1) / BN;
  // gather of tile `t` into buffer `b`: this thread owns column n0 + tid (all KP rows)
  auto issue = [&](uint32_t t, int b) {
    const uint32_t n = t * BN + tid;
    const float* src = a.win;
    bool zero = true;
    if (n < a.n_gemm) {
      uint32_t img, rem, oh, ow;
      a.fd_hw.divmod(n, img, rem);
      a.fd_wo.divmod(rem, oh, ow);
      src = a.win + static_cast<int64_t>(img) * a.img_stride + static_cast<int64_t>(oh) * a.row_stride +
            static_cast<int64_t>(ow) * a.col_stride;
      zero = false;
    }
    float* dst = Bs + b * KP * BN + tid;
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const int d = sdelta[k];
      const bool ok = d >= 0;
      cp_async_4_zfill(smem_u32(dst + k * BN), src + (ok ? d : 0), zero || !ok);
    }
    cp_async_commit();
  };
  const int tx = tid % TXN, ty = tid / TXN;
  uint32_t t = blockIdx.x;
  if (t < n_tiles) issue(t, 0);
  for (int it = 0; t < n_tiles; t += gridDim.x, ++it) {
    const int b = it & 1;
    const uint32_t tn = t + gridDim.x;
    if (tn < n_tiles) issue(tn, b ^ 1);  // its buffer was released by the barrier after compute(it-1)
    else cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    float acc[MT][MT];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < MT; ++j) acc[i][j] = 0.0f;
    const float* bs = Bs + b * KP * BN;
    // k loop to K (padded k never computed), unrolled by 4 only: a fully unrolled KP-step
    // body misses in the instruction cache (ncu: no_instruction stalls)
#pragma unroll kUnroll
    for (int kk = 0; kk < a.K; ++kk) {
      {
        float fa[MT], fb[MT];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float4 av = *reinterpret_cast<const float4*>(As + kk * BM + h * (BM / 2) + ty * 4);
          const float4 bv = *reinterpret_cast<const float4*>(bs + kk * BN + h * (BN / 2) + tx * 4);
          fa[4 * h] = av.x; fa[4 * h + 1] = av.y; fa[4 * h + 2] = av.z; fa[4 * h + 3] = av.w;
          fb[4 * h] = bv.x; fb[4 * h + 1] = bv.y; fb[4 * h + 2] = bv.z; fb[4 * h + 3] = bv.w;
        }
#pragma unroll
        for (int i = 0; i < MT; ++i) mac_row<EXACT, MT>(acc[i], fa[i], fb, a.neg_zero, a.one);
      }
    }
    __syncthreads();  // buffer b is free for the gather of tile it + 2
    // epilogue (optimized.py:209-214), overlapped with the gather in flight
    const uint32_t n0 = t * BN;
#pragma unroll
    for (int hj = 0; hj < 2; ++hj) {
      const uint32_t nq = n0 + hj * (BN / 2) + tx * 4;
      if (a.vec_out && nq + 3 < a.n_gemm) {
        uint32_t img, rem;
        a.fd_hw.divmod(nq, img, rem);
        float* base = a.out + static_cast<int64_t>(img) * a.co_out * a.hw + rem;
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const int m = (i / 4) * (BM / 2) + ty * 4 + (i % 4);
          if (m < a.M)
            __stcs(reinterpret_cast<float4*>(base + static_cast<int64_t>(m) * a.hw),
                   make_float4(acc[i][4 * hj], acc[i][4 * hj + 1], acc[i][4 * hj + 2], acc[i][4 * hj + 3]));
        }
      } else {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const uint32_t n = nq + jj;
          if (n >= a.n_gemm) continue;
          uint32_t img, rem;
          a.fd_hw.divmod(n, img, rem);
          float* base = a.out + static_cast<int64_t>(img) * a.co_out * a.hw + rem;
#pragma unroll
          for (int i = 0; i < MT; ++i) {
            const int m = (i / 4) * (BM / 2) + ty * 4 + (i % 4);
            if (m < a.M) base[static_cast<int64_t>(m) * a.hw] = acc[i][4 * hj + jj];
          }
        }
      }
    }
  }
  cp_async_wait<0>();
}

template <int KP, bool EXACT>
static cudaError_t launch_smallk(const ConvArgs& a, cudaStream_t stream) {
  const size_t smem = (static_cast<size_t>(KP) * 64 + 2ull * KP * 256) * 4 + KP * 4;
  auto kern = conv_simt_smallk_kernel<KP, EXACT>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
  if (occ < 1) occ = 1;
  const uint64_t n_tiles = (static_cast<uint64_t>(a.n_gemm) + 255) / 256;
  const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(n_tiles, static_cast<uint64_t>(occ) * sms));
  kern<<<grid, 256, smem, stream>>>(a);
  return cudaGetLastError();
}



// ---------------------------------------------------------------------------
// Tile configurations compiled into the library.
// ---------------------------------------------------------------------------
struct SimtConfig {
  int bm, bn, bk, stages;
};

constexpr int kDeltaSmemMax = IM2WIN_SIMT_SDELTA ? 48 * 1024 : 0;  // bytes of delta[] staged in smem

template <int BM, int BN, int BK, int STAGES, bool EXACT, bool VEC, int MT>
static cudaError_t launch_cfg(const ConvArgs& a0, cudaStream_t stream) {
  ConvArgs a = a0;
  a.m_tiles = (a.M - a.m_base + BM - 1) / BM;
  uint64_t n_tiles = (static_cast<uint64_t>(a.n_gemm - a.n_base) + BN - 1) / BN;
  uint64_t grid = n_tiles * a.m_tiles;
  const bool sd = static_cast<size_t>(a.Kp) * 4 <= kDeltaSmemMax;
  size_t smem = static_cast<size_t>(STAGES) * BK * (BM + BN) * 4 + (sd ? static_cast<size_t>(a.Kp) * 4 : 0);
  auto kern = sd ? conv_simt_kernel<BM, BN, BK, STAGES, EXACT, VEC, MT, true>
                 : conv_simt_kernel<BM, BN, BK, STAGES, EXACT, VEC, MT, false>;
#if IM2WIN_SIMT_BRANCHLESS && !defined(IM2WIN_SIMT_ALWAYS_PADK)
  // production toggles, 8x8 micro-tiles: a K that fills whole slabs takes the predicate-free
  // gather (measured, N=128: conv4/conv8 +2%, conv9/conv11 +2.4%; the 4x4-tile conv12 grid, one
  // barrier-bound partial wave, lost 4% with it, so 4x4 tiles keep the predicated form)
  if constexpr (STAGES > 1 && VEC && MT == 8) {
    if (a.K == a.Kp) kern = sd ? conv_simt_kernel<BM, BN, BK, STAGES, EXACT, VEC, MT, true, false>
                               : conv_simt_kernel<BM, BN, BK, STAGES, EXACT, VEC, MT, false, false>;
  }
#endif
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  im2win_note_kernel(MT == 8 ? "conv_simt_kernel (8x8 micro-tiles)" : "conv_simt_kernel (4x4 micro-tiles)");
  kern<<<static_cast<unsigned>(grid), (BM / MT) * (BN / MT), smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace im2win

using im2win::ConvArgs;

// Returns the configuration index chosen for (M, n_gemm); exposed for tests/bench.
extern "C" int im2win_simt_pick(int M, long long n_gemm, int K) {
  (void)K;
  // Measured (tools/tile_sweep.py, tools/simt_variants.py, N=128): the 64x256 8x8 tile is the
  // fastest wherever its grid fills the GPU; 96-channel layers use 96x128.  A partial last
  // wave is handled by the tail split in im2win_launch_conv_simt (conv6: 25.1 -> 26.9 TF over
  // all-4x4 tiles); only a grid under one wave that would leave the GPU under 75% busy takes
  // 4x4 micro-tiles (4x the threads): conv12 21.5 vs 17.6 TF.
  const long long slots = 148LL * 2;
  const bool m96 = M % 64 != 0 && M % 96 == 0;
  const long long ctas = m96 ? (M / 96) * ((n_gemm + 127) / 128) : ((M + 63) / 64) * ((n_gemm + 255) / 256);
  static const double below = getenv("IM2WIN_SIMT_MT4_BELOW") ? atof(getenv("IM2WIN_SIMT_MT4_BELOW")) : 0.75;
  if (ctas < slots && static_cast<double>(ctas) / static_cast<double>(slots) < below) return m96 ? 6 : 4;
  return m96 ? 2 : 1;
}

// Compiled CTA tiles (index = im2win_tile_plan.block_cfg).  0-3: 8x8 micro-tiles
// (all toggles compiled); 4-6: 4x4 micro-tiles (production toggles only).
static const int kNumCfg = 7;
static const int kBM[kNumCfg] = {128, 64, 96, 128, 64, 128, 32};
// CTA tile N extents, for reference: {128, 256, 128, 64, 64, 32, 128}
// The 64x256 tile's production kernel runs 32-deep K-slabs in 2 stages (half the slab barriers
// and loop overhead; with the packed exact pairs its body fits the instruction cache): conv4/conv8
// +0.6%, conv9 +1.3%, conv11 +2% over 16-deep slabs in 3 stages (scalar FMUL+FADD: 23 vs 30 TF).
static const int kBKc[kNumCfg] = {16, 32, 16, 16, 16, 16, 16};
static const int kMaxBK = 32;

// nchw_hw == nullptr: `win` is the im2win tensor Ĩ (row_len = Hf * w_eff).  Otherwise `win` is the
// NCHW input itself, nchw_hw = {H, W} (row_len unused): the kernels gather the same window
// elements straight from it -- Ĩ[img][c][oh][(ow*s + fw)*Hf + fh] == X[img][c][oh*s + fh][ow*s + fw]
// (layouts.py:73-83) -- so the results are bit-identical and Ĩ is never written.
int im2win_launch_conv_simt(const float* win, const float* flt, float* out, void* workspace,
                            int64_t n, int64_t c_in, int64_t c_out, int64_t h_out, int64_t w_out,
                            int64_t row_len, int h_f, int w_f, int stride, int cfg, int exact,
                            int vec, int stages, cudaStream_t stream, const char** err,
                            const int64_t* nchw_hw = nullptr) {
  using namespace im2win;
  const int64_t K = c_in * h_f * w_f;
  const int64_t hw = h_out * w_out;
  const int64_t n_gemm = n * hw;
  const int64_t img_elems = nchw_hw ? c_in * nchw_hw[0] * nchw_hw[1] : c_in * h_out * row_len;
  if (n_gemm >= (1ll << 31) || K >= (1ll << 24) || img_elems >= (1ll << 31)) {
    *err = "im2win_conv_f32: extents exceed the kernel's index range";
    return 1;
  }
  const bool auto_cfg = cfg < 0;
  if (cfg < 0) cfg = im2win_simt_pick(static_cast<int>(c_out), n_gemm, static_cast<int>(K));
  if (cfg >= kNumCfg) {
    *err = "im2win_conv_f32: unknown tile configuration";
    return 1;
  }
  if (cfg >= 4 && !(vec && stages > 1)) cfg = static_cast<int>(c_out) <= 64 ? 1 : 0;  // ablations: 8x8 tiles
  // 96-channel layers (library choice): channels 0-63 on the 64x256 tile, 64-95 on 32x128 4x4-
  // micro-tile CTAs -- both issue the packed exact pairs, which the 96x128 tile does not profit
  // from (IM2WIN_SIMT_SPLIT96=0 keeps the single 96x128 launch).  Same bits.
  const char* s96 = getenv("IM2WIN_SIMT_SPLIT96");
  const bool split96 = auto_cfg && vec && stages > 1 && cfg == 2 && c_out == 96 && IM2WIN_SIMT_FP2 &&
                       !(s96 && atoi(s96) == 0);
  const int BM = kBM[cfg], BK = split96 ? kBKc[1] : kBKc[cfg];  // K padded for every launch's slab
  const int Mp = static_cast<int>((c_out + BM - 1) / BM * BM);
  const int Kp = static_cast<int>((K + BK - 1) / BK * BK);
  if ((reinterpret_cast<uintptr_t>(workspace) & 15u) != 0) {
    *err = "im2win_conv_f32: workspace must be 16-byte aligned";
    return 1;
  }
  float* fltT = static_cast<float*>(workspace);
  int* delta = reinterpret_cast<int*>(fltT + static_cast<int64_t>(Kp) * Mp);

  if (nchw_hw)
    pack_filter_kernel<<<256, 256, 0, stream>>>(flt, fltT, delta, static_cast<int>(c_out), static_cast<int>(K), Mp,
                                                Kp, h_f, w_f, static_cast<int>(nchw_hw[0] * nchw_hw[1]),
                                                static_cast<int>(nchw_hw[1]), 1);
  else
    pack_filter_kernel<<<256, 256, 0, stream>>>(flt, fltT, delta, static_cast<int>(c_out), static_cast<int>(K), Mp,
                                                Kp, h_f, w_f, static_cast<int>(h_out * row_len), 1, h_f);
  ConvArgs a{};
  a.win = win;
  a.img_stride = static_cast<uint32_t>(img_elems);
  a.row_stride = static_cast<uint32_t>(nchw_hw ? stride * nchw_hw[1] : row_len);
  a.col_stride = static_cast<uint32_t>(nchw_hw ? stride : stride * h_f);
  a.fltT = fltT;
  a.delta = delta;
  a.out = out;
  a.M = static_cast<int>(c_out);
  a.co_out = static_cast<uint32_t>(c_out);
  a.Mp = Mp;
  a.K = static_cast<int>(K);
  a.Kp = Kp;
  a.n_gemm = static_cast<uint32_t>(n_gemm);
  a.c_in = static_cast<uint32_t>(c_in);
  a.h_out = static_cast<uint32_t>(h_out);
  a.w_out = static_cast<uint32_t>(w_out);
  a.row_len = static_cast<uint32_t>(row_len);
  a.s_hf = static_cast<uint32_t>(stride * h_f);
  a.hw = static_cast<uint32_t>(hw);
  a.fd_hw = FastDiv(static_cast<uint32_t>(hw));
  a.fd_wo = FastDiv(static_cast<uint32_t>(w_out));
  a.vec_out = (hw % 4 == 0 && (reinterpret_cast<uintptr_t>(out) & 15u) == 0) ? 1u : 0u;
  a.neg_zero = -0.0f;
  a.one = 1.0f;

  cudaError_t e = cudaSuccess;
#ifndef IM2WIN_SIMT_STAGES
#define IM2WIN_SIMT_STAGES 3
#endif
#define IM2WIN_DISPATCH(BM_, BN_, BK_)                                                              \
  if (exact && vec && stages == 3) e = launch_cfg<BM_, BN_, BK_, IM2WIN_SIMT_STAGES, true, true, 8>(a, stream); \
  else if (exact && vec && stages == 1) e = launch_cfg<BM_, BN_, BK_, 1, true, true, 8>(a, stream);  \
  else if (exact && !vec) e = launch_cfg<BM_, BN_, BK_, 3, true, false, 8>(a, stream);               \
  else if (!exact && vec) e = launch_cfg<BM_, BN_, BK_, 3, false, true, 8>(a, stream);               \
  else e = launch_cfg<BM_, BN_, BK_, 3, false, false, 8>(a, stream);
#define IM2WIN_DISPATCH4(BM_, BN_, BK_)                                                             \
  if (exact) e = launch_cfg<BM_, BN_, BK_, 3, true, true, 4>(a, stream);                            \
  else e = launch_cfg<BM_, BN_, BK_, 3, false, true, 4>(a, stream);
  // small K (conv7): the persistent kernel with a resident filter and the next tile's gather
  // in flight (library choice only; an explicit TilePlan keeps its CTA tile)
  const bool smallk = IM2WIN_SIMT_SMALLK && auto_cfg && cfg == 1 && vec && stages > 1 && c_out <= 64 && K <= 64 &&
                      (n_gemm + 255) / 256 >= 8LL * 148 * 2;
  if (smallk) {
    im2win_note_kernel("conv_simt_smallk_kernel (8x8 micro-tiles, persistent, resident filter)");
    switch (Kp) {
      case 16: e = exact ? launch_smallk<16, true>(a, stream) : launch_smallk<16, false>(a, stream); break;
      case 32: e = exact ? launch_smallk<32, true>(a, stream) : launch_smallk<32, false>(a, stream); break;
      case 48: e = exact ? launch_smallk<48, true>(a, stream) : launch_smallk<48, false>(a, stream); break;
      default: e = exact ? launch_smallk<64, true>(a, stream) : launch_smallk<64, false>(a, stream); break;
    }
  } else {
    auto dispatch = [&](int c, const ConvArgs& a) -> cudaError_t {
      cudaError_t e = cudaSuccess;
      switch (c) {
        case 0: { IM2WIN_DISPATCH(128, 128, 16) break; }
        case 1: {
          if (exact && vec && stages == 3 && IM2WIN_SIMT_FP2) e = launch_cfg<64, 256, 32, 2, true, true, 8>(a, stream);
          else { IM2WIN_DISPATCH(64, 256, 16) }
          break;
        }
        case 2: { IM2WIN_DISPATCH(96, 128, 16) break; }
        case 3: { IM2WIN_DISPATCH(128, 64, 16) break; }
        case 4: { IM2WIN_DISPATCH4(64, 64, 16) break; }
        case 5: { IM2WIN_DISPATCH4(128, 32, 16) break; }
        default: { IM2WIN_DISPATCH4(32, 128, 16) break; }
      }
      return e;
    };
    // Tail split (library choice only): when the last wave of 8x8-micro-tile CTAs would leave
    // most SMs idle, the full waves run as usual and the remaining GEMM columns go to a second
    // launch of 4x4-micro-tile CTAs (4x the CTAs, so the tail spreads over every SM).  Each
    // output is still computed by one thread over the whole K: same bits.
    int tail_cfg = -1;
    uint32_t n_main = 0;
    // (96-channel layers (cfg 2) keep one launch: their 32x128 4x4 tail measured 1.6% slower on conv1)
    if (auto_cfg && vec && stages > 1 && (cfg == 0 || cfg == 1)) {
      static thread_local int sms_cache = 0;
      if (!sms_cache) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms_cache, cudaDevAttrMultiProcessorCount, dev);
        if (sms_cache <= 0) sms_cache = 148;
      }
      const int64_t bm = kBM[cfg], bn = cfg == 1 ? 256 : 128;
      const int64_t m_t = (c_out + bm - 1) / bm, n_t = (n_gemm + bn - 1) / bn;
      const int64_t ctas = m_t * n_t, slots = 2LL * sms_cache;
      const int64_t full = ctas / slots * slots, tail = ctas - full;
      const char* te = getenv("IM2WIN_SIMT_TAIL");
      const double thr = te ? atof(te) : 0.75;
      if (full >= slots && tail > 0 && static_cast<double>(tail) < thr * static_cast<double>(slots)) {
        n_main = static_cast<uint32_t>(full / m_t * bn);
        tail_cfg = 4;
      }
    }
    if (split96) {
      ConvArgs a64 = a;
      a64.M = 64;
      e = dispatch(1, a64);
      if (e == cudaSuccess) {
        ConvArgs a32 = a;
        a32.m_base = 64;
        e = dispatch(6, a32);
        im2win_label_kernel("conv_simt_kernel (channels 0-63 on 64x256 8x8 tiles, 64-95 on 32x128 4x4 tiles)");
      }
    } else if (tail_cfg >= 0 && n_main > 0 && n_main < static_cast<uint32_t>(n_gemm)) {
      ConvArgs am = a;
      am.n_gemm = n_main;
      e = dispatch(cfg, am);
      if (e == cudaSuccess) {
        ConvArgs at = a;
        at.n_base = n_main;
        e = dispatch(tail_cfg, at);
        im2win_label_kernel("conv_simt_kernel (8x8 micro-tiles, 4x4-tile tail launch)");
      }
    } else {
      e = dispatch(cfg, a);
    }
  }
#undef IM2WIN_DISPATCH4
#undef IM2WIN_DISPATCH
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 2;
  }
  return 0;
}

// Workspace needed by im2win_launch_conv_simt for any configuration.
size_t im2win_simt_workspace_bytes(int64_t c_out, int64_t K) {
  const int64_t Mp = (c_out + 127) / 128 * 128 + 128;
  const int64_t Kp = (K + kMaxBK - 1) / kMaxBK * kMaxBK;
  return static_cast<size_t>(Kp * Mp) * 4 + static_cast<size_t>(Kp) * 4 + 256;
}

// ---------------------------------------------------------------------------
// Ablation kernel for TilePlan(micro_kernel=False) (plan.py:30-32): a 1x1
// micro-tile, one output element per thread, same staging and arithmetic.
// ---------------------------------------------------------------------------
namespace im2win {

template <int STAGES, bool EXACT>
__global__ void __launch_bounds__(256) conv_simt_1x1_kernel(const ConvArgs a) {
  constexpr int BM = 16, BN = 16, BK = 8;
  __shared__ float As[STAGES][BK][BM];
  __shared__ float Bs[STAGES][BK][BN];
  __shared__ int64_t col_off[BN];
  const int tid = threadIdx.x;
  const uint32_t m_tile = blockIdx.x % a.m_tiles;
  const uint32_t n_tile = blockIdx.x / a.m_tiles;
  const int m0 = m_tile * BM;
  const uint32_t n0 = n_tile * BN;
  if (tid < BN) {
    uint32_t n = n0 + tid;
    int64_t off = -1;
    if (n < a.n_gemm) {
      uint32_t img, rem, oh, ow;
      a.fd_hw.divmod(n, img, rem);
      a.fd_wo.divmod(rem, oh, ow);
      off = static_cast<int64_t>(img) * a.img_stride + static_cast<int64_t>(oh) * a.row_stride +
            static_cast<int64_t>(ow) * a.col_stride;
    }
    col_off[tid] = off;
  }
  __syncthreads();
  const int k_tiles = a.Kp / BK;
  auto load_stage = [&](int kt, int slot) {
    if (tid < BK * BM) {
      int r = tid / BM, c = tid % BM;
      cp_async_4(smem_u32(&As[slot][r][c]), a.fltT + static_cast<int64_t>(kt * BK + r) * a.Mp + m0 + c, 4);
    }
    if (tid < BK * BN) {
      int r = tid / BN, c = tid % BN;
      int d = __ldg(a.delta + kt * BK + r);
      int64_t co = col_off[c];
      bool ok = (d >= 0) & (co >= 0);
      cp_async_4(smem_u32(&Bs[slot][r][c]), ok ? a.win + co + d : a.win, ok ? 4u : 0u);
    }
  };
  const int ty = tid / BN, tx = tid % BN;
  float acc = 0.0f;
  auto compute_stage = [&](int slot) {
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) acc = mac<EXACT>(acc, As[slot][kk][ty], Bs[slot][kk][tx]);
  };
  if constexpr (STAGES == 1) {
    for (int kt = 0; kt < k_tiles; ++kt) {
      load_stage(kt, 0);
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      compute_stage(0);
      __syncthreads();
    }
  } else {
    load_stage(0, 0);
    cp_async_commit();
    for (int kt = 0; kt < k_tiles; ++kt) {
      if (kt + 1 < k_tiles) load_stage(kt + 1, (kt + 1) & 1);
      cp_async_commit();
      cp_async_wait<1>();
      __syncthreads();
      compute_stage(kt & 1);
      __syncthreads();
    }
  }
  const int m = m0 + ty;
  const uint32_t n = n0 + tx;
  if (m < a.M && n < a.n_gemm) {
    uint32_t img, rem;
    a.fd_hw.divmod(n, img, rem);
    a.out[static_cast<int64_t>(img) * a.co_out * a.hw + static_cast<int64_t>(m) * a.hw + rem] = acc;
  }
}

}  // namespace im2win

int im2win_launch_conv_simt_1x1(const float* win, const float* flt, float* out, void* workspace,
                                int64_t n, int64_t c_in, int64_t c_out, int64_t h_out,
                                int64_t w_out, int64_t row_len, int h_f, int w_f, int stride,
                                int exact, int stages, cudaStream_t stream, const char** err) {
  using namespace im2win;
  const int64_t K = c_in * h_f * w_f;
  const int64_t hw = h_out * w_out;
  const int64_t n_gemm = n * hw;
  if (n_gemm >= (1ll << 31) || K >= (1ll << 24) || c_in * h_out * row_len >= (1ll << 31)) {
    *err = "im2win_conv_f32: extents exceed the kernel's index range";
    return 1;
  }
  const int BM = 16, BN = 16, BK = 8;
  const int Mp = static_cast<int>((c_out + BM - 1) / BM * BM);
  const int Kp = static_cast<int>((K + BK - 1) / BK * BK);
  float* fltT = static_cast<float*>(workspace);
  int* delta = reinterpret_cast<int*>(fltT + static_cast<int64_t>(Kp) * Mp);
  pack_filter_kernel<<<256, 256, 0, stream>>>(flt, fltT, delta, static_cast<int>(c_out), static_cast<int>(K), Mp,
                                              Kp, h_f, w_f, static_cast<int>(h_out * row_len), 1, h_f);
  ConvArgs a{};
  a.win = win; a.fltT = fltT; a.delta = delta; a.out = out;
  a.img_stride = static_cast<uint32_t>(c_in * h_out * row_len);
  a.row_stride = static_cast<uint32_t>(row_len);
  a.col_stride = static_cast<uint32_t>(stride * h_f);
  a.M = static_cast<int>(c_out); a.co_out = static_cast<uint32_t>(c_out); a.Mp = Mp; a.K = static_cast<int>(K);
  a.Kp = Kp;
  a.n_gemm = static_cast<uint32_t>(n_gemm);
  a.c_in = static_cast<uint32_t>(c_in); a.h_out = static_cast<uint32_t>(h_out);
  a.w_out = static_cast<uint32_t>(w_out); a.row_len = static_cast<uint32_t>(row_len);
  a.s_hf = static_cast<uint32_t>(stride * h_f); a.hw = static_cast<uint32_t>(hw);
  a.fd_hw = FastDiv(static_cast<uint32_t>(hw)); a.fd_wo = FastDiv(static_cast<uint32_t>(w_out));
  a.m_tiles = (a.M + BM - 1) / BM;
  uint64_t grid = (static_cast<uint64_t>(n_gemm) + BN - 1) / BN * a.m_tiles;
  im2win_note_kernel("conv_simt_1x1_kernel (TilePlan micro_kernel=False)");
  if (exact) {
    if (stages > 1) conv_simt_1x1_kernel<2, true><<<static_cast<unsigned>(grid), 256, 0, stream>>>(a);
    else conv_simt_1x1_kernel<1, true><<<static_cast<unsigned>(grid), 256, 0, stream>>>(a);
  } else {
    if (stages > 1) conv_simt_1x1_kernel<2, false><<<static_cast<unsigned>(grid), 256, 0, stream>>>(a);
    else conv_simt_1x1_kernel<1, false><<<static_cast<unsigned>(grid), 256, 0, stream>>>(a);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { *err = cudaGetErrorString(e); return 2; }
  return 0;
}

// ---------------------------------------------------------------------------
// Paper Alg. 2 "basic" im2win kernel (winconv
// _basic_window_kernel, reference.py:180-206): grid (N/32, M/32), block 32x32,
// one output per thread, operands read straight from global memory through the
// window map Ĩ[n, c, oh, (ow*s + fw)*Hf + fh] -- no shared-memory tiling, no
// register micro-tile.  Same unfused ascending-k arithmetic (bit-exact); it is the
// baseline the tiled kernel is measured against (reference test_acceptance.py:185-215).
// ---------------------------------------------------------------------------
namespace im2win {

__global__ void __launch_bounds__(1024) conv_basic_kernel(const float* __restrict__ win, const float* __restrict__ flt,
                                                          float* __restrict__ out, uint32_t n_gemm, uint32_t M,
                                                          uint32_t K, uint32_t c_in, uint32_t h_out, uint32_t row_len,
                                                          uint32_t h_f, uint32_t w_f, uint32_t s_hf, FastDiv fd_hw,
                                                          FastDiv fd_wo, uint32_t hw) {
  const uint32_t n = blockIdx.x * 32 + threadIdx.x;
  const uint32_t m = blockIdx.y * 32 + threadIdx.y;
  if (n >= n_gemm || m >= M) return;
  uint32_t img, rem, oh, ow;
  fd_hw.divmod(n, img, rem);
  fd_wo.divmod(rem, oh, ow);
  const float* wp = win + (static_cast<int64_t>(img) * c_in * h_out + oh) * row_len + static_cast<int64_t>(ow) * s_hf;
  const float* fp = flt + static_cast<int64_t>(m) * K;
  const int64_t chan = static_cast<int64_t>(h_out) * row_len;
  float acc = 0.0f;
  uint32_t k = 0;
  for (uint32_t c = 0; c < c_in; ++c) {
    for (uint32_t fh = 0; fh < h_f; ++fh) {
      for (uint32_t fw = 0; fw < w_f; ++fw, ++k) acc = __fadd_rn(acc, __fmul_rn(__ldg(fp + k), __ldg(wp + fw * h_f + fh)));
    }
    wp += chan;
  }
  out[static_cast<int64_t>(img) * M * hw + static_cast<int64_t>(m) * hw + rem] = acc;
}

}  // namespace im2win

int im2win_launch_conv_basic(const float* win, const float* flt, float* out, int64_t n, int64_t c_in, int64_t c_out,
                             int64_t h_out, int64_t w_out, int64_t row_len, int h_f, int w_f, int stride,
                             cudaStream_t stream, const char** err) {
  using namespace im2win;
  const int64_t hw = h_out * w_out, n_gemm = n * hw, K = c_in * h_f * w_f;
  if (n_gemm >= (1ll << 31) || (n_gemm + 31) / 32 >= (1ll << 31) || (c_out + 31) / 32 > 65535) {
    *err = "im2win_conv_basic_f32: extents exceed the kernel's index range";
    return 1;
  }
  dim3 grid(static_cast<unsigned>((n_gemm + 31) / 32), static_cast<unsigned>((c_out + 31) / 32));
  im2win_note_kernel("conv_basic_kernel (paper Alg. 2)");
  conv_basic_kernel<<<grid, dim3(32, 32), 0, stream>>>(
      win, flt, out, static_cast<uint32_t>(n_gemm), static_cast<uint32_t>(c_out), static_cast<uint32_t>(K),
      static_cast<uint32_t>(c_in), static_cast<uint32_t>(h_out), static_cast<uint32_t>(row_len), h_f, w_f,
      static_cast<uint32_t>(stride * h_f), FastDiv(static_cast<uint32_t>(hw)), FastDiv(static_cast<uint32_t>(w_out)),
      static_cast<uint32_t>(hw));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 2;
  }
  return 0;
}
