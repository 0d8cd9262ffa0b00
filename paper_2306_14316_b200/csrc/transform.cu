// im2win transform: NCHW input -> window-ordered tensor (N, C, Ho, Hf*w_eff).
//
// Restates winconv `_im2win_fill` (reference pkg/src/winconv/layouts.py:73-83):
//     dst[i, r, m, c*Hf + u] = src[i, r, m*s + u, c]      c < w_eff, u < Hf
// as an HBM-bound, bit-exact copy.  Design (B200):
//   * the output is one flat contiguous array of G = N*C*Ho rows of RL = Hf*w_eff
//     floats; a CTA owns R consecutive output rows (possibly spanning several
//     (image, channel) planes) and therefore one contiguous output range;
//   * the input rows those output rows read form one contiguous range of input
//     rows; they are staged once into shared memory with coalesced loads
//     (each input row feeds ceil(Hf/s) output rows, so HBM reads it once);
//   * the output range is written with aligned 16-byte stores, the (c, u)
//     decode of each element stepped incrementally from one fast division.
#include "common.cuh"

namespace im2win {

struct TransformArgs {
  const float* __restrict__ src;
  float* __restrict__ dst;
  uint32_t rows_total;  // G = N*C*Ho
  uint32_t h_out, h_in, w_in, stride, h_f, w_eff, row_len;
  uint32_t pitch;       // smem row pitch (floats), odd to spread banks
  uint32_t rows_per_cta;
  FastDiv fd_ho, fd_rl, fd_hf, fd_weff;
};

IM2WIN_DEVICE uint64_t in_row_of(const TransformArgs& a, uint32_t g) {
  uint32_t plane, m;
  a.fd_ho.divmod(g, plane, m);
  return static_cast<uint64_t>(plane) * a.h_in + static_cast<uint64_t>(m) * a.stride;
}

__global__ void __launch_bounds__(256) im2win_transform_kernel(const TransformArgs a) {
  extern __shared__ float smem[];
  const uint32_t g0 = blockIdx.x * a.rows_per_cta;
  const uint32_t nrows_out = min(a.rows_per_cta, a.rows_total - g0);
  int* rowoff = reinterpret_cast<int*>(smem);           // [rows_per_cta]
  float* tile = smem + ((a.rows_per_cta + 3) & ~3u);    // [span][pitch]

  const uint64_t r_lo = in_row_of(a, g0);
  const uint64_t r_hi = in_row_of(a, g0 + nrows_out - 1) + a.h_f;
  const uint32_t nrows_in = static_cast<uint32_t>(r_hi - r_lo);

  for (uint32_t gl = threadIdx.x; gl < nrows_out; gl += blockDim.x)
    rowoff[gl] = static_cast<int>(in_row_of(a, g0 + gl) - r_lo) * static_cast<int>(a.pitch);

  // ---- stage input rows [r_lo, r_hi), columns [0, w_eff) ----
  {
    const float* src = a.src + r_lo * a.w_in;
    const uint32_t total = nrows_in * a.w_eff;
    constexpr int U = 4;
    uint32_t idx = threadIdx.x;
    for (; idx + (U - 1) * blockDim.x < total; idx += U * blockDim.x) {
      float v[U];
      uint32_t so[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        uint32_t row, col;
        a.fd_weff.divmod(idx + q * blockDim.x, row, col);
        v[q] = __ldcs(src + static_cast<uint64_t>(row) * a.w_in + col);
        so[q] = row * a.pitch + col;
      }
#pragma unroll
      for (int q = 0; q < U; ++q) tile[so[q]] = v[q];
    }
    for (; idx < total; idx += blockDim.x) {
      uint32_t row, col;
      a.fd_weff.divmod(idx, row, col);
      tile[row * a.pitch + col] = __ldcs(src + static_cast<uint64_t>(row) * a.w_in + col);
    }
  }
  __syncthreads();

  // ---- write the contiguous output range [g0*RL, (g0+nrows_out)*RL) ----
  const uint64_t e_begin = static_cast<uint64_t>(g0) * a.row_len;
  const uint32_t count = nrows_out * a.row_len;
  float* dst = a.dst + e_begin;
  const uint32_t head = min(count, static_cast<uint32_t>((4u - (e_begin & 3u)) & 3u));
  const uint32_t nvec = (count - head) >> 2;

  auto value_at = [&](uint32_t e) -> float {
    uint32_t gl, j, c, u;
    a.fd_rl.divmod(e, gl, j);
    a.fd_hf.divmod(j, c, u);
    return tile[rowoff[gl] + u * a.pitch + c];
  };

  if (threadIdx.x < head) dst[threadIdx.x] = value_at(threadIdx.x);
  {
    const uint32_t tail_begin = head + nvec * 4;
    const uint32_t t = tail_begin + threadIdx.x;
    if (t < count) dst[t] = value_at(t);
  }
  float4* dst4 = reinterpret_cast<float4*>(dst + head);
  for (uint32_t vi = threadIdx.x; vi < nvec; vi += blockDim.x) {
    uint32_t e = head + vi * 4;
    uint32_t gl, j, c, u;
    a.fd_rl.divmod(e, gl, j);
    a.fd_hf.divmod(j, c, u);
    int base = rowoff[gl];
    float out[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      out[q] = tile[base + u * a.pitch + c];
      ++u;
      ++j;
      if (u == a.h_f) { u = 0; ++c; }
      if (j == a.row_len) { j = 0; c = 0; u = 0; ++gl; if (q < 3) base = rowoff[gl]; }
    }
    dst4[vi] = make_float4(out[0], out[1], out[2], out[3]);
  }
}

// Host planning: rows per CTA and the worst-case input-row span.
struct TransformPlan {
  uint32_t rows_per_cta;
  uint32_t span;
  uint32_t pitch;
  size_t smem_bytes;
  uint32_t grid;
};

static uint64_t host_in_row(uint64_t g, uint64_t h_out, uint64_t h_in, uint64_t s) {
  return (g / h_out) * h_in + (g % h_out) * s;
}

static uint32_t host_span(uint32_t R, uint32_t h_out, uint32_t h_in, uint32_t s, uint32_t h_f) {
  // span of input rows read by output rows [p, p+R) maximised over the phase p.
  uint64_t best = 0;
  for (uint32_t p = 0; p < h_out; ++p) {
    uint64_t lo = host_in_row(p, h_out, h_in, s);
    uint64_t hi = host_in_row(p + R - 1, h_out, h_in, s) + h_f;
    if (hi - lo > best) best = hi - lo;
  }
  return static_cast<uint32_t>(best);
}

static TransformPlan plan_transform(uint32_t rows_total, uint32_t h_out, uint32_t h_in, uint32_t s,
                                    uint32_t h_f, uint32_t w_eff, uint32_t row_len, size_t smem_cap) {
  TransformPlan p{};
  p.pitch = w_eff | 1u;
  uint32_t R = (8192 + row_len - 1) / row_len;
  uint32_t min_r = (2 * h_f + s - 1) / s;
  if (R < min_r) R = min_r;
  if (R > rows_total) R = rows_total;
  if (R < 1) R = 1;
  for (;;) {
    p.span = host_span(R, h_out, h_in, s, h_f);
    p.smem_bytes = (static_cast<size_t>((R + 3) & ~3u) + static_cast<size_t>(p.span) * p.pitch) * 4;
    if (p.smem_bytes <= smem_cap || R == 1) break;
    R = R / 2;
  }
  p.rows_per_cta = R;
  p.grid = (rows_total + R - 1) / R;
  return p;
}

}  // namespace im2win

// Launcher used by the C ABI (capi.cu).
int im2win_launch_transform(const float* src, float* dst, int64_t n, int64_t c, int64_t h, int64_t w,
                            int h_f, int w_f, int stride, int64_t h_out, int64_t w_eff,
                            cudaStream_t stream, const char** err) {
  using namespace im2win;
  const int64_t rows_total = n * c * h_out;
  const int64_t row_len = static_cast<int64_t>(h_f) * w_eff;
  if (rows_total >= (1ll << 31) || row_len >= (1ll << 24) || n * c * h >= (1ll << 31)) {
    *err = "im2win_transform_f32: extents exceed the 31-bit row index range";
    return 1;
  }
  const size_t smem_cap = 96 * 1024;
  TransformPlan p = plan_transform(static_cast<uint32_t>(rows_total), static_cast<uint32_t>(h_out),
                                   static_cast<uint32_t>(h), static_cast<uint32_t>(stride),
                                   static_cast<uint32_t>(h_f), static_cast<uint32_t>(w_eff),
                                   static_cast<uint32_t>(row_len), smem_cap);
  if (p.smem_bytes > smem_cap) {
    *err = "im2win_transform_f32: one output row needs more shared memory than available";
    return 1;
  }
  TransformArgs a;
  a.src = src;
  a.dst = dst;
  a.rows_total = static_cast<uint32_t>(rows_total);
  a.h_out = static_cast<uint32_t>(h_out);
  a.h_in = static_cast<uint32_t>(h);
  a.w_in = static_cast<uint32_t>(w);
  a.stride = static_cast<uint32_t>(stride);
  a.h_f = static_cast<uint32_t>(h_f);
  a.w_eff = static_cast<uint32_t>(w_eff);
  a.row_len = static_cast<uint32_t>(row_len);
  a.pitch = p.pitch;
  a.rows_per_cta = p.rows_per_cta;
  a.fd_ho = FastDiv(a.h_out);
  a.fd_rl = FastDiv(a.row_len);
  a.fd_hf = FastDiv(a.h_f);
  a.fd_weff = FastDiv(a.w_eff);
  (void)w_f;
  if (p.smem_bytes > 48 * 1024) {
    cudaFuncSetAttribute(im2win_transform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem_cap));
  }
  im2win_transform_kernel<<<p.grid, 256, p.smem_bytes, stream>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 2;
  }
  return 0;
}
