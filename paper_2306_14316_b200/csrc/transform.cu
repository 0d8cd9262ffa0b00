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
  uint32_t tile_floats; // staged-input capacity (floats, multiple of 4)
  uint32_t rows_per_cta;
  FastDiv fd_ho, fd_rl, fd_hf, fd_weff;
};

IM2WIN_DEVICE uint64_t in_row_of(const TransformArgs& a, uint32_t g) {
  uint32_t plane, m;
  a.fd_ho.divmod(g, plane, m);
  return static_cast<uint64_t>(plane) * a.h_in + static_cast<uint64_t>(m) * a.stride;
}

__global__ void __launch_bounds__(256) im2win_transform_kernel(const TransformArgs a) {
  extern __shared__ __align__(16) float smem[];
  const uint32_t g0 = blockIdx.x * a.rows_per_cta;
  const uint32_t nrows_out = min(a.rows_per_cta, a.rows_total - g0);
  int* rowoff = reinterpret_cast<int*>(smem);                     // [rows_per_cta]
  float* tile = smem + ((a.rows_per_cta + 3) & ~3u);              // staged input, pitch w_in
  float* obuf = tile + a.tile_floats;                              // output chunk (+3 slack)

  const uint64_t r_lo = in_row_of(a, g0);
  const uint64_t r_hi = in_row_of(a, g0 + nrows_out - 1) + a.h_f;

  // ---- phase 1: stage input rows [r_lo, r_hi) as one flat range (all w_in columns) ----
  // Aligned 16-byte loads; the smem image is shifted so aligned global float4s land on
  // aligned smem float4s (tile[i + tshift] holds flat element i).
  const uint64_t f_begin = r_lo * a.w_in;
  const uint32_t f_count = static_cast<uint32_t>((r_hi - r_lo) * a.w_in);
  const float* src = a.src + f_begin;
  const uint32_t f_head = min(f_count, static_cast<uint32_t>((4u - (f_begin & 3u)) & 3u));
  const uint32_t tshift = (4u - f_head) & 3u;
  {
    const uint32_t nvec = (f_count - f_head) >> 2;
    const float4* src4 = reinterpret_cast<const float4*>(src + f_head);
    float4* t4 = reinterpret_cast<float4*>(tile + tshift + f_head);
    constexpr int U = 4;
    uint32_t v = threadIdx.x;
    for (; v + (U - 1) * blockDim.x < nvec; v += U * blockDim.x) {
      float4 r[U];
#pragma unroll
      for (int q = 0; q < U; ++q) r[q] = __ldcs(src4 + v + q * blockDim.x);
#pragma unroll
      for (int q = 0; q < U; ++q) t4[v + q * blockDim.x] = r[q];
    }
    for (; v < nvec; v += blockDim.x) t4[v] = __ldcs(src4 + v);
    if (threadIdx.x < f_head) tile[tshift + threadIdx.x] = __ldcs(src + threadIdx.x);
    const uint32_t tail = f_head + (nvec << 2);
    if (tail + threadIdx.x < f_count) tile[tshift + tail + threadIdx.x] = __ldcs(src + tail + threadIdx.x);
  }
  for (uint32_t gl = threadIdx.x; gl < nrows_out; gl += blockDim.x)
    rowoff[gl] = static_cast<int>((in_row_of(a, g0 + gl) - r_lo) * a.w_in + tshift);

  // ---- phase 2: build the output chunk in smem ----
  // item = (output row gl, source column c); it writes the h_f values of that
  // column: out[gl*RL + c*Hf + u] = in[row(gl) + u][c].  Lanes take consecutive
  // columns: reads hit consecutive banks, writes stride Hf (odd -> conflict free).
  const uint64_t e_begin = static_cast<uint64_t>(g0) * a.row_len;
  const uint32_t count = nrows_out * a.row_len;
  const uint32_t head = min(count, static_cast<uint32_t>((4u - (e_begin & 3u)) & 3u));
  const uint32_t oshift = (4u - head) & 3u;
  __syncthreads();
  {
    const uint32_t items = nrows_out * a.w_eff;
    for (uint32_t it = threadIdx.x; it < items; it += blockDim.x) {
      uint32_t gl, c;
      a.fd_weff.divmod(it, gl, c);
      const float* tp = tile + rowoff[gl] + c;
      float* op = obuf + oshift + gl * a.row_len + c * a.h_f;
      for (uint32_t u = 0; u < a.h_f; ++u) op[u] = tp[u * a.w_in];
    }
  }
  __syncthreads();

  // ---- phase 3: stream the chunk out with aligned 16-byte stores ----
  float* dst = a.dst + e_begin;
  const uint32_t nvec = (count - head) >> 2;
  if (threadIdx.x < head) dst[threadIdx.x] = obuf[oshift + threadIdx.x];
  const uint32_t tail = head + (nvec << 2);
  if (tail + threadIdx.x < count) dst[tail + threadIdx.x] = obuf[oshift + tail + threadIdx.x];
  const float4* o4 = reinterpret_cast<const float4*>(obuf + oshift + head);
  float4* d4 = reinterpret_cast<float4*>(dst + head);
  for (uint32_t v = threadIdx.x; v < nvec; v += blockDim.x) __stcs(d4 + v, o4[v]);
}

// Host planning: rows per CTA and the worst-case input-row span.
struct TransformPlan {
  uint32_t rows_per_cta;
  uint32_t span;
  uint32_t tile_floats;
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

static TransformPlan plan_transform(uint32_t rows_total, uint32_t h_out, uint32_t h_in, uint32_t w_in,
                                    uint32_t s, uint32_t h_f, uint32_t row_len, size_t smem_cap) {
  TransformPlan p{};
  uint32_t R = (8192 + row_len - 1) / row_len;
  uint32_t min_r = (2 * h_f + s - 1) / s;
  if (R < min_r) R = min_r;
  if (R > rows_total) R = rows_total;
  if (R < 1) R = 1;
  for (;;) {
    p.span = host_span(R, h_out, h_in, s, h_f);
    p.tile_floats = (p.span * w_in + 3 + 3) & ~3u;
    const size_t out_floats = static_cast<size_t>(R) * row_len + 3;
    p.smem_bytes = (static_cast<size_t>((R + 3) & ~3u) + p.tile_floats + out_floats) * 4;
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
                                   static_cast<uint32_t>(h), static_cast<uint32_t>(w), static_cast<uint32_t>(stride),
                                   static_cast<uint32_t>(h_f), static_cast<uint32_t>(row_len), smem_cap);
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
  a.tile_floats = p.tile_floats;
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
