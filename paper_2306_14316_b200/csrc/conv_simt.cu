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
#include "common.cuh"

namespace im2win {

struct ConvArgs {
  const float* __restrict__ win;    // im2win tensor, flat
  const float* __restrict__ fltT;   // packed filter [Kp][Mp]
  const int* __restrict__ delta;    // [Kp], -1 beyond K
  float* __restrict__ out;          // (N, Co, Ho, Wo)
  int M, Mp, K, Kp;
  uint32_t n_gemm;                  // N*Ho*Wo
  uint32_t c_in, h_out, w_out, row_len, s_hf, hw;
  FastDiv fd_hw, fd_wo;
  uint32_t m_tiles;
};

// ---------------------------------------------------------------------------
// pack: FT[k][m] = F[m][k] (zero padded), delta[k] = c*Ho*RL + fw*Hf + fh
// ---------------------------------------------------------------------------
__global__ void pack_filter_kernel(const float* __restrict__ flt, float* __restrict__ fltT,
                                   int* __restrict__ delta, int M, int K, int Mp, int Kp, int h_f,
                                   int w_f, int chan_stride) {
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
        d = c * chan_stride + fw * h_f + fh;
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

template <int BM, int BN, int BK, int STAGES, bool EXACT, bool VEC, bool MB = false>
__global__ void __launch_bounds__((BM / 8) * (BN / 8), 2)
    conv_simt_kernel(const ConvArgs a) {
  constexpr int NT = (BM / 8) * (BN / 8);
  constexpr int TXN = BN / 8;                 // threads along n
  constexpr int CPT = (BN + NT - 1) / NT;     // gather columns per thread
  static_assert(BK % 4 == 0, "BK must be a multiple of 4 (int4 delta loads)");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* As = reinterpret_cast<float*>(smem_raw);  // [STAGES][BK][BM]
  float* Bs = As + STAGES * BK * BM;               // [STAGES][BK][BN]

  const int tid = threadIdx.x;
  const uint32_t m_tile = blockIdx.x % a.m_tiles;
  const uint32_t n_tile = blockIdx.x / a.m_tiles;
  const int m0 = m_tile * BM;
  const uint32_t n0 = n_tile * BN;

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
      bsrc[j] = a.win + (static_cast<int64_t>(img) * a.c_in * a.h_out + oh) * a.row_len +
                static_cast<int64_t>(ow) * a.s_hf;
      bzero[j] = false;
    }
  }

  const int k_tiles = a.Kp / BK;
  const int k_full = a.K / BK;  // slabs with no padded k

  auto load_stage = [&](int kt, int slot) {
    // filter slab: BK rows of BM floats, 16-byte copies
    const float* fsrc = a.fltT + static_cast<int64_t>(kt) * BK * a.Mp + m0;
    float* adst = As + slot * BK * BM;
#pragma unroll
    for (int q = tid; q < BK * BM / 4; q += NT) {
      int r = q / (BM / 4), c4 = q % (BM / 4);
      cp_async_16(smem_u32(adst + r * BM + c4 * 4), fsrc + static_cast<int64_t>(r) * a.Mp + c4 * 4, 16);
    }
    // window slab: each gathering thread owns whole columns of BK elements
    int d[BK];
#pragma unroll
    for (int q = 0; q < BK / 4; ++q) {
      int4 v = __ldg(reinterpret_cast<const int4*>(a.delta + kt * BK) + q);
      d[4 * q] = v.x; d[4 * q + 1] = v.y; d[4 * q + 2] = v.z; d[4 * q + 3] = v.w;
    }
    float* bdst = Bs + slot * BK * BN;
    const bool full = kt < k_full;
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int c = tid + j * NT;
      if (c < BN) {
        if (full) {
#pragma unroll
          for (int kk = 0; kk < BK; ++kk) cp_async_4_zfill(smem_u32(bdst + kk * BN + c), bsrc[j] + d[kk], bzero[j]);
        } else {
#pragma unroll
          for (int kk = 0; kk < BK; ++kk) {
            const bool ok = d[kk] >= 0;
            cp_async_4_zfill(smem_u32(bdst + kk * BN + c), ok ? bsrc[j] + d[kk] : a.win, bzero[j] || !ok);
          }
        }
      }
    }
  };

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;

  const int tx = tid % TXN;
  const int ty = tid / TXN;

  auto compute_stage = [&](int slot) {
    const float* as = As + slot * BK * BM;
    const float* bs = Bs + slot * BK * BN;
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float fa[8], fb[8];
      if constexpr (VEC) {
        float4 a0 = *reinterpret_cast<const float4*>(as + kk * BM + ty * 4);
        float4 a1 = *reinterpret_cast<const float4*>(as + kk * BM + BM / 2 + ty * 4);
        float4 b0 = *reinterpret_cast<const float4*>(bs + kk * BN + tx * 4);
        float4 b1 = *reinterpret_cast<const float4*>(bs + kk * BN + BN / 2 + tx * 4);
        fa[0] = a0.x; fa[1] = a0.y; fa[2] = a0.z; fa[3] = a0.w;
        fa[4] = a1.x; fa[5] = a1.y; fa[6] = a1.z; fa[7] = a1.w;
        fb[0] = b0.x; fb[1] = b0.y; fb[2] = b0.z; fb[3] = b0.w;
        fb[4] = b1.x; fb[5] = b1.y; fb[6] = b1.z; fb[7] = b1.w;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          fa[i] = as[kk * BM + ty * 4 + i];
          fa[4 + i] = as[kk * BM + BM / 2 + ty * 4 + i];
          fb[i] = bs[kk * BN + tx * 4 + i];
          fb[4 + i] = bs[kk * BN + BN / 2 + tx * 4 + i];
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = mac<EXACT>(acc[i][j], fa[i], fb[j]);
    }
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
  } else if constexpr (MB) {
    // mbarrier ring: full[s] completes when every thread's copies for the slab in
    // slot s have landed (cp.async.mbarrier.arrive.noinc); empty[s] when every warp
    // has consumed it.  No CTA-wide barrier in the K loop: warps may drift up to
    // STAGES-PD-1 slabs apart.  PD+1 slabs are in flight ahead of the consumer.
    constexpr int PD = STAGES - 3;
    __shared__ __align__(8) uint64_t full_bar[STAGES];
    __shared__ __align__(8) uint64_t empty_bar[STAGES];
    if (tid == 0) {
#pragma unroll
      for (int s = 0; s < STAGES; ++s) {
        mbarrier_init(&full_bar[s], NT);
        mbarrier_init(&empty_bar[s], NT / 32);
      }
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s <= PD; ++s) {
      if (s < k_tiles) {
        load_stage(s, s);
        cp_async_arrive_noinc(&full_bar[s]);
      }
    }
    for (int kt = 0; kt < k_tiles; ++kt) {
      const int pf = kt + PD + 1;
      if (pf < k_tiles) {
        const int ps = pf % STAGES;
        if (pf >= STAGES) mbarrier_wait_parity(&empty_bar[ps], ((pf - STAGES) / STAGES) & 1);
        load_stage(pf, ps);
        cp_async_arrive_noinc(&full_bar[ps]);
      }
      const int slot = kt % STAGES;
      mbarrier_wait_parity(&full_bar[slot], (kt / STAGES) & 1);
      compute_stage(slot);
      __syncwarp();
      if ((tid & 31) == 0) mbarrier_arrive(&empty_bar[slot]);
    }
  } else {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < k_tiles) load_stage(s, s);
      cp_async_commit();
    }
    for (int kt = 0; kt < k_tiles; ++kt) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      int pf = kt + STAGES - 1;
      if (pf < k_tiles) load_stage(pf, pf % STAGES);
      cp_async_commit();
      compute_stage(kt % STAGES);
    }
  }

  // epilogue: scatter to NCHW (optimized.py:209-214)
  int64_t dst_off[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint32_t n = n0 + (j < 4 ? tx * 4 + j : BN / 2 + tx * 4 + (j - 4));
    int64_t off = -1;
    if (n < a.n_gemm) {
      uint32_t img, rem;
      a.fd_hw.divmod(n, img, rem);
      off = static_cast<int64_t>(img) * a.M * a.hw + rem;
    }
    dst_off[j] = off;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int m = m0 + (i < 4 ? ty * 4 + i : BM / 2 + ty * 4 + (i - 4));
    if (m < a.M) {
      int64_t mo = static_cast<int64_t>(m) * a.hw;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (dst_off[j] >= 0) a.out[dst_off[j] + mo] = acc[i][j];
    }
  }
}

// ---------------------------------------------------------------------------
// Tile configurations compiled into the library.
// ---------------------------------------------------------------------------
struct SimtConfig {
  int bm, bn, bk, stages;
};

template <int BM, int BN, int BK, int STAGES, bool EXACT, bool VEC, bool MB = false>
static cudaError_t launch_cfg(const ConvArgs& a0, cudaStream_t stream) {
  ConvArgs a = a0;
  a.m_tiles = (a.M + BM - 1) / BM;
  uint64_t n_tiles = (static_cast<uint64_t>(a.n_gemm) + BN - 1) / BN;
  uint64_t grid = n_tiles * a.m_tiles;
  size_t smem = static_cast<size_t>(STAGES) * BK * (BM + BN) * 4;
  auto kern = conv_simt_kernel<BM, BN, BK, STAGES, EXACT, VEC, MB>;
  if (smem + 1024 > 48 * 1024) {  // + static smem (mbarriers)
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  kern<<<static_cast<unsigned>(grid), (BM / 8) * (BN / 8), smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace im2win

using im2win::ConvArgs;

// Returns the configuration index chosen for (M, n_gemm); exposed for tests/bench.
extern "C" int im2win_simt_pick(int M, long long n_gemm, int K) {
  (void)K;
  if (M <= 64) return 1;    // 64 x 256
  if (M <= 96) return 2;    // 96 x 128
  if (n_gemm < 148LL * 128 * 2) return 3;  // 128 x 64 for small-N layers (wave fill)
  return 0;                 // 128 x 128
}

// Compiled CTA tiles (index = im2win_tile_plan.block_cfg).  0-3 are the
// production tiles (all toggles compiled); 4+ are exploration tiles.
static const int kNumCfg = 7;
static const int kBM[kNumCfg] = {128, 64, 96, 128, 64, 128, 64};
static const int kBN[kNumCfg] = {128, 256, 128, 64, 256, 128, 256};
static const int kBKc[kNumCfg] = {16, 16, 16, 16, 16, 16, 16};
static const int kMaxBK = 32;

int im2win_launch_conv_simt(const float* win, const float* flt, float* out, void* workspace,
                            int64_t n, int64_t c_in, int64_t c_out, int64_t h_out, int64_t w_out,
                            int64_t row_len, int h_f, int w_f, int stride, int cfg, int exact,
                            int vec, int stages, cudaStream_t stream, const char** err) {
  using namespace im2win;
  const int64_t K = c_in * h_f * w_f;
  const int64_t hw = h_out * w_out;
  const int64_t n_gemm = n * hw;
  if (n_gemm >= (1ll << 31) || K >= (1ll << 24) || c_in * h_out * row_len >= (1ll << 31)) {
    *err = "im2win_conv_f32: extents exceed the kernel's index range";
    return 1;
  }
  if (cfg < 0) cfg = im2win_simt_pick(static_cast<int>(c_out), n_gemm, static_cast<int>(K));
  if (cfg >= kNumCfg) {
    *err = "im2win_conv_f32: unknown tile configuration";
    return 1;
  }
  if (cfg >= 4 && !(exact && vec && stages > 1)) cfg = im2win_simt_pick(static_cast<int>(c_out), n_gemm, static_cast<int>(K));
  const int BM = kBM[cfg], BK = kBKc[cfg];
  const int Mp = static_cast<int>((c_out + BM - 1) / BM * BM);
  const int Kp = static_cast<int>((K + BK - 1) / BK * BK);
  float* fltT = static_cast<float*>(workspace);
  int* delta = reinterpret_cast<int*>(fltT + static_cast<int64_t>(Kp) * Mp);

  pack_filter_kernel<<<256, 256, 0, stream>>>(flt, fltT, delta, static_cast<int>(c_out), static_cast<int>(K), Mp,
                                              Kp, h_f, w_f, static_cast<int>(h_out * row_len));
  ConvArgs a{};
  a.win = win;
  a.fltT = fltT;
  a.delta = delta;
  a.out = out;
  a.M = static_cast<int>(c_out);
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

  cudaError_t e = cudaSuccess;
#define IM2WIN_DISPATCH(BM_, BN_, BK_)                                                              \
  if (exact && vec && stages == 3) e = launch_cfg<BM_, BN_, BK_, 3, true, true>(a, stream);          \
  else if (exact && vec && stages == 1) e = launch_cfg<BM_, BN_, BK_, 1, true, true>(a, stream);     \
  else if (exact && !vec) e = launch_cfg<BM_, BN_, BK_, 3, true, false>(a, stream);                  \
  else if (!exact && vec) e = launch_cfg<BM_, BN_, BK_, 3, false, true>(a, stream);               \
  else e = launch_cfg<BM_, BN_, BK_, 3, false, false>(a, stream);
  switch (cfg) {
    case 0: { IM2WIN_DISPATCH(128, 128, 16) break; }
    case 1: { IM2WIN_DISPATCH(64, 256, 16) break; }
    case 2: { IM2WIN_DISPATCH(96, 128, 16) break; }
    case 3: { IM2WIN_DISPATCH(128, 64, 16) break; }
    case 4: e = launch_cfg<64, 256, 16, 4, true, true, true>(a, stream); break;   // mbarrier ring (explored)
    case 5: e = launch_cfg<128, 128, 16, 4, true, true, true>(a, stream); break;  // mbarrier ring (explored)
    case 6: e = launch_cfg<64, 256, 16, 5, true, true, true>(a, stream); break;  // deeper mbarrier ring
    default: *err = "im2win_conv_f32: unknown tile configuration"; return 1;
  }
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
  constexpr int BM = 16, BN = 16, BK = 8, NT = 256;
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
      off = (static_cast<int64_t>(img) * a.c_in * a.h_out + oh) * a.row_len + static_cast<int64_t>(ow) * a.s_hf;
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
    a.out[static_cast<int64_t>(img) * a.M * a.hw + static_cast<int64_t>(m) * a.hw + rem] = acc;
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
                                              Kp, h_f, w_f, static_cast<int>(h_out * row_len));
  ConvArgs a{};
  a.win = win; a.fltT = fltT; a.delta = delta; a.out = out;
  a.M = static_cast<int>(c_out); a.Mp = Mp; a.K = static_cast<int>(K); a.Kp = Kp;
  a.n_gemm = static_cast<uint32_t>(n_gemm);
  a.c_in = static_cast<uint32_t>(c_in); a.h_out = static_cast<uint32_t>(h_out);
  a.w_out = static_cast<uint32_t>(w_out); a.row_len = static_cast<uint32_t>(row_len);
  a.s_hf = static_cast<uint32_t>(stride * h_f); a.hw = static_cast<uint32_t>(hw);
  a.fd_hw = FastDiv(static_cast<uint32_t>(hw)); a.fd_wo = FastDiv(static_cast<uint32_t>(w_out));
  a.m_tiles = (a.M + BM - 1) / BM;
  uint64_t grid = (static_cast<uint64_t>(n_gemm) + BN - 1) / BN * a.m_tiles;
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
