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
#include <algorithm>
#include <cstdlib>

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
  uint32_t pad;         // zero padding on every side (pipelined kernel only); h_out/w_eff are padded geometry
  uint32_t src_mis, dst_mis;  // (ptr % 16) / 4 of src / dst: the staged kernel aligns its float4s to the address
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
  const uint32_t f_head = min(f_count, static_cast<uint32_t>((4u - ((f_begin + a.src_mis) & 3u)) & 3u));
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
  const uint32_t head = min(count, static_cast<uint32_t>((4u - ((e_begin + a.dst_mis) & 3u)) & 3u));
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

// ---------------------------------------------------------------------------
// Pipelined persistent variant (the production path).
//
// Same chunking as above (a chunk = R consecutive output rows = one contiguous
// output range; its input rows = one contiguous input range), but each CTA
// walks chunks blockIdx.x, +gridDim.x, ... with two shared-memory stages:
//   * the input range of chunk j+1 is fetched by one TMA bulk copy
//     (cp.async.bulk, mbarrier complete_tx) while chunk j is being built;
//   * the built output range of chunk j leaves by one TMA bulk store
//     (cp.async.bulk.global.shared::cta, bulk_group) that drains while chunk
//     j+1 is built; its buffer is reused two chunks later after
//     cp.async.bulk.wait_group.read.
// Unaligned input/output ends (< 16 B) are moved with plain loads/stores.
// Needs 16 B aligned src/dst base pointers (checked by the launcher).
// ---------------------------------------------------------------------------
constexpr uint32_t kXformThreads = 256;

struct PipeArgs {
  TransformArgs t;
  uint64_t src_floats;   // total input elements (bulk loads never read past it)
  uint32_t n_chunks;
  uint32_t obuf_floats;  // per stage, multiple of 4
  uint32_t rowoff_ints;  // per stage, multiple of 4
};

IM2WIN_DEVICE void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
IM2WIN_DEVICE void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
IM2WIN_DEVICE void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
IM2WIN_DEVICE void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
IM2WIN_DEVICE void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

IM2WIN_DEVICE int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
IM2WIN_DEVICE int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

struct ChunkGeom {
  uint32_t g0, nrows;
  uint64_t r_lo, f_begin, f_end, a_begin, a_end;
};

// Real input rows [lo, hi) that output row g reads (padded rows outside [0, H) are zeros).
IM2WIN_DEVICE uint64_t in_row_lo(const TransformArgs& a, uint32_t g) {
  uint32_t plane, m;
  a.fd_ho.divmod(g, plane, m);
  const int64_t r = static_cast<int64_t>(m) * a.stride - a.pad;
  return static_cast<uint64_t>(plane) * a.h_in + static_cast<uint64_t>(imin64(imax64(r, 0), a.h_in));
}
IM2WIN_DEVICE uint64_t in_row_hi(const TransformArgs& a, uint32_t g) {
  uint32_t plane, m;
  a.fd_ho.divmod(g, plane, m);
  const int64_t r = static_cast<int64_t>(m) * a.stride - a.pad + a.h_f;
  return static_cast<uint64_t>(plane) * a.h_in + static_cast<uint64_t>(imin64(imax64(r, 0), a.h_in));
}

IM2WIN_DEVICE ChunkGeom chunk_geom(const PipeArgs& p, uint32_t chunk) {
  const TransformArgs& a = p.t;
  ChunkGeom c;
  c.g0 = chunk * a.rows_per_cta;
  c.nrows = min(a.rows_per_cta, a.rows_total - c.g0);
  c.r_lo = in_row_lo(a, c.g0);
  const uint64_t r_hi = in_row_hi(a, c.g0 + c.nrows - 1);
  c.f_begin = c.r_lo * a.w_in;
  c.f_end = r_hi * a.w_in;
  c.a_begin = c.f_begin & ~3ull;
  c.a_end = min((c.f_end + 3) & ~3ull, p.src_floats & ~3ull);
  return c;
}

// Build one output chunk in shared memory.  Items (row gl, column col) are
// strided by the CTA size; (gl, col) advances incrementally (no division in
// the loop).  HF > 0 unrolls the Hf copies (loads first, then stores).
// PAD: ro[gl] is the staged offset of padded row m*s - p, column -p (may point before
// the tile); uv[gl] packs the valid tap range [u_lo, u_hi) of that output row.  A value
// is read only when its row tap and column are inside the real input, else it is +0.
template <int HF, bool PAD>
IM2WIN_DEVICE void build_chunk(const TransformArgs& a, const float* __restrict__ tb, const int* __restrict__ ro,
                               const uint32_t* __restrict__ uv, float* __restrict__ ob, uint32_t nrows, uint32_t tid,
                               uint32_t dg, uint32_t dc) {
  const uint32_t w_eff = a.w_eff, w_in = a.w_in, row_len = a.row_len;
  const uint32_t items = nrows * w_eff;
  uint32_t gl, col;
  a.fd_weff.divmod(tid, gl, col);
  for (uint32_t it = tid; it < items; it += kXformThreads) {
    const float* tp = tb + ro[gl] + static_cast<int>(col);
    if constexpr (PAD) {
      const uint32_t u_lo = uv[gl] & 0xffffu, u_hi = uv[gl] >> 16;
      const bool col_ok = col >= a.pad && col < a.pad + w_in;
      if constexpr (HF > 0) {
        float* op = ob + gl * row_len + col * HF;
        float v[HF];
#pragma unroll
        for (int u = 0; u < HF; ++u)
          v[u] = (col_ok && static_cast<uint32_t>(u) >= u_lo && static_cast<uint32_t>(u) < u_hi)
                     ? tp[static_cast<int>(u * w_in)] : 0.0f;
#pragma unroll
        for (int u = 0; u < HF; ++u) op[u] = v[u];
      } else {
        const uint32_t hf = a.h_f;
        float* op = ob + gl * row_len + col * hf;
        for (uint32_t u = 0; u < hf; ++u)
          op[u] = (col_ok && u >= u_lo && u < u_hi) ? tp[static_cast<int>(u * w_in)] : 0.0f;
      }
    } else if constexpr (HF > 0) {
      float* op = ob + gl * row_len + col * HF;
      float v[HF];
#pragma unroll
      for (int u = 0; u < HF; ++u) v[u] = tp[u * w_in];
#pragma unroll
      for (int u = 0; u < HF; ++u) op[u] = v[u];
    } else {
      const uint32_t hf = a.h_f;
      float* op = ob + gl * row_len + col * hf;
      for (uint32_t u = 0; u < hf; ++u) op[u] = tp[u * w_in];
    }
    col += dc;
    gl += dg;
    if (col >= w_eff) {
      col -= w_eff;
      ++gl;
    }
  }
}

template <int HF, bool PAD>
__global__ void __launch_bounds__(kXformThreads) im2win_transform_pipe_kernel(const PipeArgs p) {
  const TransformArgs& a = p.t;
  uint32_t dg, dc;  // kXformThreads = dg * w_eff + dc
  a.fd_weff.divmod(kXformThreads, dg, dc);
  extern __shared__ __align__(16) float smem[];
  __shared__ __align__(8) uint64_t full[2];
  int* rowoff = reinterpret_cast<int*>(smem);          // [2][rowoff_ints] (+ [2][rowoff_ints] tap ranges if PAD)
  uint32_t* urange = reinterpret_cast<uint32_t*>(rowoff + 2 * p.rowoff_ints);
  float* tile = smem + (PAD ? 4 : 2) * p.rowoff_ints;  // [2][tile_floats]
  float* obuf = tile + 2 * a.tile_floats;               // [2][obuf_floats]
  const uint32_t tid = threadIdx.x;

  if (tid == 0) {
    mbarrier_init(&full[0], 1);
    mbarrier_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](uint32_t chunk, int b) {
    const ChunkGeom c = chunk_geom(p, chunk);
    const uint32_t bytes = c.a_end > c.a_begin ? static_cast<uint32_t>(c.a_end - c.a_begin) * 4u : 0u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&full[b])), "r"(bytes)
                 : "memory");
    if (bytes) bulk_load(tile + b * a.tile_floats, a.src + c.a_begin, bytes, &full[b]);
  };

  uint32_t chunk = blockIdx.x;
  if (tid == 0 && chunk < p.n_chunks) issue(chunk, 0);
  for (uint32_t j = 0; chunk < p.n_chunks; chunk += gridDim.x, ++j) {
    const int b = j & 1;
    const uint32_t next = chunk + gridDim.x;
    // stage b^1 was last read by chunk j-1's build, which ended at a CTA barrier
    if (tid == 0 && next < p.n_chunks) issue(next, b ^ 1);

    const ChunkGeom c = chunk_geom(p, chunk);
    float* tb = tile + b * a.tile_floats;
    float* ob = obuf + b * p.obuf_floats;
    int* ro = rowoff + b * p.rowoff_ints;
    uint32_t* uv = urange + b * p.rowoff_ints;
    const uint32_t tshift = static_cast<uint32_t>(c.f_begin - c.a_begin);
    for (uint32_t gl = tid; gl < c.nrows; gl += blockDim.x) {
      if constexpr (PAD) {
        uint32_t plane, m;
        a.fd_ho.divmod(c.g0 + gl, plane, m);
        const int64_t top = static_cast<int64_t>(m) * a.stride - a.pad;  // real row of tap u = 0
        const int64_t row0 = static_cast<int64_t>(plane) * a.h_in + top - static_cast<int64_t>(c.r_lo);
        ro[gl] = static_cast<int>(row0 * a.w_in - a.pad + tshift);
        const int64_t u_lo = imax64(0, -top), u_hi = imin64(a.h_f, static_cast<int64_t>(a.h_in) - top);
        uv[gl] = static_cast<uint32_t>(u_lo) | (static_cast<uint32_t>(imax64(u_hi, u_lo)) << 16);
      } else {
        ro[gl] = static_cast<int>((in_row_of(a, c.g0 + gl) - c.r_lo) * a.w_in + tshift);
      }
    }

    mbarrier_wait_parity(&full[b], (j >> 1) & 1);
    // input tail the bulk copy could not cover (end of the tensor, < 4 floats)
    for (uint64_t f = max(c.a_end, c.a_begin) + tid; f < c.f_end; f += blockDim.x)
      tb[f - c.a_begin] = a.src[f];
    // the bulk store of chunk j-2 read this stage's obuf; keep only chunk j-1's in flight
    if (tid == 0) bulk_wait_read<1>();
    __syncthreads();

    // build: item = (row gl, column col) writes Hf values (conflict-free, see above)
    const uint64_t e_begin = static_cast<uint64_t>(c.g0) * a.row_len;
    const uint32_t count = c.nrows * a.row_len;
    const uint32_t head = min(count, static_cast<uint32_t>((4u - (e_begin & 3u)) & 3u));
    const uint32_t oshift = (4u - head) & 3u;
    build_chunk<HF, PAD>(a, tb, ro, uv, ob + oshift, c.nrows, tid, dg, dc);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();

    float* dst = a.dst + e_begin;
    const uint32_t nvec = (count - head) >> 2;
    const uint32_t tail = head + (nvec << 2);
    if (tid < head) dst[tid] = ob[oshift + tid];
    if (tail + tid < count) dst[tail + tid] = ob[oshift + tail + tid];
    if (tid == 0) {
      if (nvec) bulk_store(dst + head, ob + oshift + head, nvec * 16u);
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait_all();
}

// Host planning: rows per CTA and the worst-case input-row span.
struct TransformPlan {
  uint32_t rows_per_cta;
  uint32_t span;
  uint32_t tile_floats;
  size_t smem_bytes;
  uint32_t grid;
};


// Real input rows [lo, hi) of output row g with zero padding `pad` (pad = 0: hi = lo + h_f).
static uint64_t host_row_lo(uint64_t g, uint64_t h_out, uint64_t h_in, uint64_t s, uint64_t pad) {
  const int64_t r = static_cast<int64_t>((g % h_out) * s) - static_cast<int64_t>(pad);
  return (g / h_out) * h_in + static_cast<uint64_t>(std::min<int64_t>(std::max<int64_t>(r, 0), h_in));
}
static uint64_t host_row_hi(uint64_t g, uint64_t h_out, uint64_t h_in, uint64_t s, uint64_t h_f, uint64_t pad) {
  const int64_t r = static_cast<int64_t>((g % h_out) * s + h_f) - static_cast<int64_t>(pad);
  return (g / h_out) * h_in + static_cast<uint64_t>(std::min<int64_t>(std::max<int64_t>(r, 0), h_in));
}

static uint32_t host_span(uint32_t R, uint32_t h_out, uint32_t h_in, uint32_t s, uint32_t h_f, uint32_t pad = 0) {
  // span of input rows read by output rows [p, p+R) maximised over the phase p.
  uint64_t best = 0;
  for (uint32_t p = 0; p < h_out; ++p) {
    uint64_t lo = host_row_lo(p, h_out, h_in, s, pad);
    uint64_t hi = host_row_hi(p + R - 1, h_out, h_in, s, h_f, pad);
    if (hi > lo && hi - lo > best) best = hi - lo;
  }
  return static_cast<uint32_t>(best);
}

static TransformPlan plan_transform(uint32_t rows_total, uint32_t h_out, uint32_t h_in, uint32_t w_in,
                                    uint32_t s, uint32_t h_f, uint32_t row_len, size_t smem_cap,
                                    uint32_t target_floats = 8192, uint32_t pad = 0) {
  TransformPlan p{};
  uint32_t R = (target_floats + row_len - 1) / row_len;
  uint32_t min_r = (2 * h_f + s - 1) / s;
  if (R < min_r) R = min_r;
  if (R > rows_total) R = rows_total;
  if (R < 1) R = 1;
  for (;;) {
    p.span = host_span(R, h_out, h_in, s, h_f, pad);
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
                            int h_f, int w_f, int stride, int64_t h_out, int64_t w_eff, int pad,
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
  a.pad = static_cast<uint32_t>(pad);
  a.src_mis = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(src) & 15u) >> 2);
  a.dst_mis = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(dst) & 15u) >> 2);
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 3u) != 0) {
    *err = "im2win_transform_f32: buffers must be 4-byte aligned";
    return 1;
  }
  (void)w_f;
  const bool aligned = (reinterpret_cast<uintptr_t>(src) & 15u) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0;
  // pipelined path: two stages of (row offsets, staged input, output chunk)
  const char* tgt_env = getenv("IM2WIN_XFORM_CHUNK");
  const uint32_t target = tgt_env ? static_cast<uint32_t>(atoi(tgt_env)) : 4096u;
  TransformPlan q = plan_transform(static_cast<uint32_t>(rows_total), static_cast<uint32_t>(h_out),
                                   static_cast<uint32_t>(h), static_cast<uint32_t>(w), static_cast<uint32_t>(stride),
                                   static_cast<uint32_t>(h_f), static_cast<uint32_t>(row_len), 48 * 1024, target,
                                   static_cast<uint32_t>(pad));
  PipeArgs pa;
  pa.t = a;
  pa.t.rows_per_cta = q.rows_per_cta;
  pa.t.tile_floats = (q.span * static_cast<uint32_t>(w) + 4 + 3) & ~3u;
  pa.obuf_floats = (q.rows_per_cta * static_cast<uint32_t>(row_len) + 4 + 3) & ~3u;
  pa.rowoff_ints = (q.rows_per_cta + 3) & ~3u;
  pa.src_floats = static_cast<uint64_t>(n * c * h * w);
  pa.n_chunks = q.grid;
  const size_t pipe_smem = 2ull * ((pad ? 2 : 1) * pa.rowoff_ints + pa.t.tile_floats + pa.obuf_floats) * 4;
  if (pad && !(aligned && pipe_smem <= 200 * 1024)) {
    *err = "im2win_transform_f32: zero padding needs 16-byte aligned buffers";
    return 1;
  }
  if (aligned && pipe_smem <= 200 * 1024) {
    void (*kern)(const PipeArgs) = im2win_transform_pipe_kernel<0, false>;
    int ki = 0;
    switch (h_f) {
      case 3: kern = pad ? im2win_transform_pipe_kernel<3, true> : im2win_transform_pipe_kernel<3, false>; ki = 1; break;
      case 5: kern = pad ? im2win_transform_pipe_kernel<5, true> : im2win_transform_pipe_kernel<5, false>; ki = 2; break;
      case 7: kern = pad ? im2win_transform_pipe_kernel<7, true> : im2win_transform_pipe_kernel<7, false>; ki = 3; break;
      case 11: kern = pad ? im2win_transform_pipe_kernel<11, true> : im2win_transform_pipe_kernel<11, false>; ki = 4; break;
      default: kern = pad ? im2win_transform_pipe_kernel<0, true> : im2win_transform_pipe_kernel<0, false>; break;
    }
    ki += pad ? 8 : 0;
    // per-(kernel, smem size) occupancy cache: keeps host work per call small
    static thread_local struct { int dev, ki; size_t smem; int occ; int sms; } cache[8];
    static thread_local int cache_n = 0;
    int occ = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    for (int i = 0; i < cache_n; ++i)
      if (cache[i].dev == dev && cache[i].ki == ki && cache[i].smem == pipe_smem) {
        occ = cache[i].occ;
        sms = cache[i].sms;
      }
    if (!occ) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kXformThreads, pipe_smem);
      if (occ < 1) occ = 1;
      cache[cache_n < 8 ? cache_n : 7] = {dev, ki, pipe_smem, occ, sms};
      if (cache_n < 8) ++cache_n;
    }
    const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(pa.n_chunks, static_cast<uint64_t>(sms) * occ));
    kern<<<grid, kXformThreads, pipe_smem, stream>>>(pa);
  } else {
    if (p.smem_bytes > 48 * 1024) {
      cudaFuncSetAttribute(im2win_transform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem_cap));
    }
    im2win_transform_kernel<<<p.grid, 256, p.smem_bytes, stream>>>(a);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = cudaGetErrorString(e);
    return 2;
  }
  return 0;
}
