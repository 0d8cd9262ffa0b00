#include <atomic>
// extern "C" boundary of libim2win_sm100.so (declared in include/im2win_sm100.h).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/im2win_sm100.h"

int im2win_launch_transform(const float* src, float* dst, int64_t n, int64_t c, int64_t h, int64_t w,
                            int h_f, int w_f, int stride, int64_t h_out, int64_t w_eff, int pad,
                            cudaStream_t stream, const char** err);
int im2win_launch_conv_simt(const float* win, const float* flt, float* out, void* workspace,
                            int64_t n, int64_t c_in, int64_t c_out, int64_t h_out, int64_t w_out,
                            int64_t row_len, int h_f, int w_f, int stride, int cfg, int exact,
                            int vec, int stages, cudaStream_t stream, const char** err,
                            const int64_t* nchw_hw = nullptr);
int im2win_launch_conv_simt_1x1(const float* win, const float* flt, float* out, void* workspace,
                                int64_t n, int64_t c_in, int64_t c_out, int64_t h_out,
                                int64_t w_out, int64_t row_len, int h_f, int w_f, int stride,
                                int exact, int stages, cudaStream_t stream, const char** err);
size_t im2win_simt_workspace_bytes(int64_t c_out, int64_t K);
size_t im2win_tc_workspace_bytes(int64_t c_out, int64_t K, int variant);
int im2win_launch_conv_tc(const float* win, const float* flt, float* out, void* workspace,
                          int64_t n, int64_t c_in, int64_t c_out, int64_t h_out, int64_t w_out,
                          int64_t row_len, int h_f, int w_f, int stride, int variant, int cfg,
                          cudaStream_t stream, const char** err);

static thread_local char g_last_error[512] = "";

static int fail(int code, const char* msg) {
  snprintf(g_last_error, sizeof(g_last_error), "%s", msg ? msg : "unknown error");
  return code;
}

// The library links its own (static) CUDA runtime, whose current-device state
// is independent of the caller's.  Every entry point therefore makes the
// device that owns the output buffer current before launching.
static int bind_device_of(const void* ptr) {
  cudaPointerAttributes attr;
  cudaError_t e = cudaPointerGetAttributes(&attr, ptr);
  if (e != cudaSuccess) return fail(2, cudaGetErrorString(e));
  if (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged)
    return fail(1, "pointer is not device memory");
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != attr.device) {
    e = cudaSetDevice(attr.device);
    if (e != cudaSuccess) return fail(2, cudaGetErrorString(e));
  }
  return 0;
}

int im2win_set_error(int code, const char* msg) { return fail(code, msg); }

static thread_local const char* g_last_kernel = "";
static std::atomic<long long> g_conv_launches{0};
// every conv kernel launch site reports its kernel here (once per launch)
void im2win_note_kernel(const char* name) {
  g_last_kernel = name;
  g_conv_launches.fetch_add(1, std::memory_order_relaxed);
}
void im2win_label_kernel(const char* name) { g_last_kernel = name; }

extern "C" {

const char* im2win_last_error(void) { return g_last_error; }

const char* im2win_last_kernel(void) { return g_last_kernel; }

int64_t im2win_conv_launch_count(void) { return g_conv_launches.load(std::memory_order_relaxed); }

int32_t im2win_abi_version(void) { return 100; }

int im2win_transform_f32_padded(const float* src, float* dst, int64_t n, int64_t c, int64_t h, int64_t w,
                                int32_t h_f, int32_t w_f, int32_t stride, int32_t pad, void* stream) {
  g_last_error[0] = '\0';
  if (!src || !dst) return fail(1, "im2win_transform_f32: null pointer");
  if (n < 1 || c < 1 || h < 1 || w < 1 || h_f < 1 || w_f < 1 || stride < 1 || pad < 0)
    return fail(1, "im2win_transform_f32: extents must be positive (pad >= 0)");
  if (h_f > h + 2 * pad || w_f > w + 2 * pad) return fail(1, "im2win_transform_f32: filter larger than input");
  if (int rc = bind_device_of(dst)) return rc;
  const int64_t h_out = (h + 2 * pad - h_f) / stride + 1;
  const int64_t w_out = (w + 2 * pad - w_f) / stride + 1;
  const int64_t w_eff = (w_out - 1) * stride + w_f;
  const char* err = nullptr;
  int rc = im2win_launch_transform(src, dst, n, c, h, w, h_f, w_f, stride, h_out, w_eff, pad,
                                   static_cast<cudaStream_t>(stream), &err);
  return rc ? fail(rc, err) : 0;
}

int im2win_transform_f32(const float* src, float* dst, int64_t n, int64_t c, int64_t h, int64_t w,
                         int32_t h_f, int32_t w_f, int32_t stride, void* stream) {
  return im2win_transform_f32_padded(src, dst, n, c, h, w, h_f, w_f, stride, 0, stream);
}

size_t im2win_conv_workspace_bytes(int64_t c_in, int64_t c_out, int32_t h_f, int32_t w_f,
                                   int32_t variant) {
  const int64_t K = c_in * h_f * w_f;
  if (variant == IM2WIN_TF32 || variant == IM2WIN_BF16) return im2win_tc_workspace_bytes(c_out, K, variant);
  return im2win_simt_workspace_bytes(c_out, K);
}

int im2win_conv_f32(const float* windows, const float* flt, float* out, int64_t n, int64_t c_in,
                    int64_t c_out, int64_t h_out, int64_t w_out, int64_t row_len, int32_t h_f,
                    int32_t w_f, int32_t stride, const im2win_tile_plan* plan, int32_t variant,
                    void* workspace, size_t workspace_bytes, void* stream) {
  g_last_error[0] = '\0';
  if (!windows || !flt || !out) return fail(1, "im2win_conv_f32: null pointer");
  if (n < 1 || c_in < 1 || c_out < 1 || h_out < 1 || w_out < 1 || h_f < 1 || w_f < 1 || stride < 1)
    return fail(1, "im2win_conv_f32: extents must be positive");
  const int64_t w_eff = (w_out - 1) * stride + w_f;
  if (row_len != h_f * w_eff) return fail(1, "im2win_conv_f32: row_len != h_f * w_eff");
  if (workspace_bytes < im2win_conv_workspace_bytes(c_in, c_out, h_f, w_f, variant) || !workspace)
    return fail(1, "im2win_conv_f32: workspace too small");
  if (int rc = bind_device_of(out)) return rc;
  im2win_tile_plan def = {-1, 1, 1, 1};
  const im2win_tile_plan* p = plan ? plan : &def;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* err = nullptr;
  int rc = 0;
  switch (variant) {
    case IM2WIN_FP32_EXACT:
    case IM2WIN_FP32_FMA: {
      const int exact = variant == IM2WIN_FP32_EXACT;
      const int stages = p->prefetch_double_buffer ? 3 : 1;
      if (!p->micro_kernel)
        rc = im2win_launch_conv_simt_1x1(windows, flt, out, workspace, n, c_in, c_out, h_out, w_out,
                                         row_len, h_f, w_f, stride, exact, stages, st, &err);
      else
        rc = im2win_launch_conv_simt(windows, flt, out, workspace, n, c_in, c_out, h_out, w_out,
                                     row_len, h_f, w_f, stride, p->block_cfg, exact,
                                     p->vectorized_load, stages, st, &err);
      break;
    }
    case IM2WIN_TF32:
    case IM2WIN_BF16:
      rc = im2win_launch_conv_tc(windows, flt, out, workspace, n, c_in, c_out, h_out, w_out, row_len,
                                 h_f, w_f, stride, variant, p->block_cfg, st, &err);
      break;
    default:
      return fail(1, "im2win_conv_f32: unknown variant");
  }
  return rc ? fail(rc, err) : 0;
}

int im2win_conv_nchw_f32(const float* x, const float* flt, float* out, int64_t n, int64_t c_in, int64_t h,
                         int64_t w, int64_t c_out, int32_t h_f, int32_t w_f, int32_t stride,
                         const im2win_tile_plan* plan, int32_t variant, void* workspace, size_t workspace_bytes,
                         void* stream) {
  g_last_error[0] = '\0';
  if (!x || !flt || !out) return fail(1, "im2win_conv_nchw_f32: null pointer");
  if (n < 1 || c_in < 1 || c_out < 1 || h < 1 || w < 1 || h_f < 1 || w_f < 1 || stride < 1)
    return fail(1, "im2win_conv_nchw_f32: extents must be positive");
  if (h_f > h || w_f > w) return fail(1, "im2win_conv_nchw_f32: filter larger than input");
  if (variant != IM2WIN_FP32_EXACT && variant != IM2WIN_FP32_FMA)
    return fail(1, "im2win_conv_nchw_f32: variant must be IM2WIN_FP32_EXACT or IM2WIN_FP32_FMA");
  if (workspace_bytes < im2win_conv_workspace_bytes(c_in, c_out, h_f, w_f, variant) || !workspace)
    return fail(1, "im2win_conv_nchw_f32: workspace too small");
  im2win_tile_plan def = {-1, 1, 1, 1};
  const im2win_tile_plan* p = plan ? plan : &def;
  if (!p->micro_kernel) return fail(1, "im2win_conv_nchw_f32: micro_kernel=False is an ablation of the Ĩ path");
  if (int rc = bind_device_of(out)) return rc;
  const int64_t h_out = (h - h_f) / stride + 1, w_out = (w - w_f) / stride + 1;
  const int64_t hw[2] = {h, w};
  const char* err = nullptr;
  const int rc = im2win_launch_conv_simt(x, flt, out, workspace, n, c_in, c_out, h_out, w_out, 0, h_f, w_f, stride,
                                         p->block_cfg, variant == IM2WIN_FP32_EXACT, p->vectorized_load,
                                         p->prefetch_double_buffer ? 3 : 1, static_cast<cudaStream_t>(stream), &err,
                                         hw);
  return rc ? fail(rc, err) : 0;
}

}  // extern "C"

// ---- tensor-core fast path over the channels-innermost window layout (conv_tc_cl.cu) ----
int im2win_launch_transform_cl(const float* src, void* dst, int64_t n, int64_t c, int64_t h, int64_t w, int h_f,
                               int w_f, int stride, int bf16, cudaStream_t stream, const char** err);
size_t im2win_tc_cl_workspace_bytes(int64_t c_out, int64_t K);
int im2win_launch_conv_tc_cl(const void* win_cl, const float* flt, float* out, void* workspace, int64_t n,
                             int64_t c_in, int64_t c_out, int64_t h_out, int64_t w_out, int h_f, int w_f, int stride,
                             int bf16, cudaStream_t stream, const char** err);

extern "C" {

int im2win_transform_cl(const float* src, void* dst, int64_t n, int64_t c, int64_t h, int64_t w, int32_t h_f,
                        int32_t w_f, int32_t stride, int32_t dtype, void* stream) {
  g_last_error[0] = '\0';
  if (!src || !dst) return fail(1, "im2win_transform_cl: null pointer");
  if (n < 1 || c < 1 || h < 1 || w < 1 || h_f < 1 || w_f < 1 || stride < 1)
    return fail(1, "im2win_transform_cl: extents must be positive");
  if (h_f > h || w_f > w) return fail(1, "im2win_transform_cl: filter larger than input");
  if (dtype != 0 && dtype != 1) return fail(1, "im2win_transform_cl: dtype must be 0 (f32) or 1 (bf16)");
  if (int rc = bind_device_of(dst)) return rc;
  const char* err = nullptr;
  int rc = im2win_launch_transform_cl(src, dst, n, c, h, w, h_f, w_f, stride, dtype, static_cast<cudaStream_t>(stream),
                                      &err);
  return rc ? fail(rc, err) : 0;
}

size_t im2win_conv_cl_workspace_bytes(int64_t c_in, int64_t c_out, int32_t h_f, int32_t w_f) {
  return im2win_tc_cl_workspace_bytes(c_out, c_in * h_f * w_f);
}

int im2win_conv_cl(const void* windows_cl, const float* flt, float* out, int64_t n, int64_t c_in, int64_t c_out,
                   int64_t h_out, int64_t w_out, int32_t h_f, int32_t w_f, int32_t stride, int32_t variant,
                   void* workspace, size_t workspace_bytes, void* stream) {
  g_last_error[0] = '\0';
  if (!windows_cl || !flt || !out || !workspace) return fail(1, "im2win_conv_cl: null pointer");
  if (n < 1 || c_in < 1 || c_out < 1 || h_out < 1 || w_out < 1 || h_f < 1 || w_f < 1 || stride < 1)
    return fail(1, "im2win_conv_cl: extents must be positive");
  if (variant != IM2WIN_TF32 && variant != IM2WIN_BF16)
    return fail(1, "im2win_conv_cl: variant must be IM2WIN_TF32 or IM2WIN_BF16");
  if (workspace_bytes < im2win_conv_cl_workspace_bytes(c_in, c_out, h_f, w_f))
    return fail(1, "im2win_conv_cl: workspace too small");
  if (int rc = bind_device_of(out)) return rc;
  const char* err = nullptr;
  int rc = im2win_launch_conv_tc_cl(windows_cl, flt, out, workspace, n, c_in, c_out, h_out, w_out, h_f, w_f, stride,
                                    variant == IM2WIN_BF16, static_cast<cudaStream_t>(stream), &err);
  return rc ? fail(rc, err) : 0;
}

}  // extern "C"

// ---- fused tensor-core path: TMA window view over an NHWC copy (conv_tc_fused.cu) ----
int im2win_launch_nchw_to_nhwc(const float* src, void* dst, int64_t n, int64_t c, int64_t h, int64_t w, int bf16,
                               int pad, cudaStream_t stream, const char** err);
size_t im2win_tc_fused_workspace_bytes(int64_t c_in, int64_t c_out, int h_f, int w_f);
int im2win_launch_conv_tc_fused(const void* x_cl, const float* flt, float* out, void* workspace, int64_t n,
                                int64_t c_in, int64_t h, int64_t w, int64_t c_out, int h_f, int w_f, int stride,
                                int bf16, const float* feed_src, cudaStream_t stream, const char** err);
size_t im2win_tc_fused_feed_workspace_bytes(int64_t n, int64_t c_in, int64_t c_out, int h_f, int w_f);

extern "C" {

int im2win_nchw_to_nhwc_padded(const float* src, void* dst, int64_t n, int64_t c, int64_t h, int64_t w, int32_t dtype,
                               int32_t pad, void* stream) {
  g_last_error[0] = '\0';
  if (!src || !dst) return fail(1, "im2win_nchw_to_nhwc: null pointer");
  if (n < 1 || c < 1 || h < 1 || w < 1 || pad < 0) return fail(1, "im2win_nchw_to_nhwc: extents must be positive");
  if (dtype != 0 && dtype != 1) return fail(1, "im2win_nchw_to_nhwc: dtype must be 0 (f32) or 1 (bf16)");
  if (pad > 0 && (reinterpret_cast<uintptr_t>(dst) & 15) != 0)
    return fail(1, "im2win_nchw_to_nhwc: a padded copy needs a 16-byte aligned destination");
  if (int rc = bind_device_of(dst)) return rc;
  const char* err = nullptr;
  int rc = im2win_launch_nchw_to_nhwc(src, dst, n, c, h, w, dtype, pad, static_cast<cudaStream_t>(stream), &err);
  return rc ? fail(rc, err) : 0;
}

int im2win_nchw_to_nhwc(const float* src, void* dst, int64_t n, int64_t c, int64_t h, int64_t w, int32_t dtype,
                        void* stream) {
  return im2win_nchw_to_nhwc_padded(src, dst, n, c, h, w, dtype, 0, stream);
}

size_t im2win_conv_fused_workspace_bytes(int64_t c_in, int64_t c_out, int32_t h_f, int32_t w_f) {
  return im2win_tc_fused_workspace_bytes(c_in, c_out, h_f, w_f);
}

int im2win_conv_fused(const void* x_nhwc, const float* flt, float* out, int64_t n, int64_t c_in, int64_t h,
                      int64_t w, int64_t c_out, int32_t h_f, int32_t w_f, int32_t stride, int32_t variant,
                      void* workspace, size_t workspace_bytes, void* stream) {
  g_last_error[0] = '\0';
  if (!x_nhwc || !flt || !out || !workspace) return fail(1, "im2win_conv_fused: null pointer");
  if (n < 1 || c_in < 1 || c_out < 1 || h < 1 || w < 1 || h_f < 1 || w_f < 1 || stride < 1)
    return fail(1, "im2win_conv_fused: extents must be positive");
  if (h_f > h || w_f > w) return fail(1, "im2win_conv_fused: filter larger than input");
  if (variant != IM2WIN_TF32 && variant != IM2WIN_BF16)
    return fail(1, "im2win_conv_fused: variant must be IM2WIN_TF32 or IM2WIN_BF16");
  if (workspace_bytes < im2win_conv_fused_workspace_bytes(c_in, c_out, h_f, w_f))
    return fail(1, "im2win_conv_fused: workspace too small");
  if (int rc = bind_device_of(out)) return rc;
  const char* err = nullptr;
  int rc = im2win_launch_conv_tc_fused(x_nhwc, flt, out, workspace, n, c_in, h, w, c_out, h_f, w_f, stride,
                                       variant == IM2WIN_BF16, nullptr, static_cast<cudaStream_t>(stream), &err);
  return rc ? fail(rc, err) : 0;
}

size_t im2win_conv_fused_nchw_workspace_bytes(int64_t n, int64_t c_in, int64_t c_out, int32_t h_f, int32_t w_f) {
  return im2win_tc_fused_feed_workspace_bytes(n, c_in, c_out, h_f, w_f);
}

int im2win_conv_fused_nchw(const float* x, void* x_nhwc, const float* flt, float* out, int64_t n, int64_t c_in,
                           int64_t h, int64_t w, int64_t c_out, int32_t h_f, int32_t w_f, int32_t stride,
                           int32_t variant, void* workspace, size_t workspace_bytes, void* stream) {
  g_last_error[0] = '\0';
  if (!x || !x_nhwc || !flt || !out || !workspace) return fail(1, "im2win_conv_fused_nchw: null pointer");
  if (n < 1 || c_in < 1 || c_out < 1 || h < 1 || w < 1 || h_f < 1 || w_f < 1 || stride < 1)
    return fail(1, "im2win_conv_fused_nchw: extents must be positive");
  if (h_f > h || w_f > w) return fail(1, "im2win_conv_fused_nchw: filter larger than input");
  if (variant != IM2WIN_TF32 && variant != IM2WIN_BF16)
    return fail(1, "im2win_conv_fused_nchw: variant must be IM2WIN_TF32 or IM2WIN_BF16");
  if (workspace_bytes < im2win_conv_fused_nchw_workspace_bytes(n, c_in, c_out, h_f, w_f))
    return fail(1, "im2win_conv_fused_nchw: workspace too small");
  if ((reinterpret_cast<uintptr_t>(x_nhwc) & 15) != 0 || (reinterpret_cast<uintptr_t>(workspace) & 15) != 0)
    return fail(1, "im2win_conv_fused_nchw: x_nhwc and workspace must be 16-byte aligned");
  if (int rc = bind_device_of(out)) return rc;
  const char* err = nullptr;
  int rc = im2win_launch_conv_tc_fused(x_nhwc, flt, out, workspace, n, c_in, h, w, c_out, h_f, w_f, stride,
                                       variant == IM2WIN_BF16, x, static_cast<cudaStream_t>(stream), &err);
  return rc ? fail(rc, err) : 0;
}

}  // extern "C"

// ---- paper Alg. 2 basic kernel (reference compute_from_windows_basic, reference.py:180-219) ----
int im2win_launch_conv_basic(const float* win, const float* flt, float* out, int64_t n, int64_t c_in, int64_t c_out,
                             int64_t h_out, int64_t w_out, int64_t row_len, int h_f, int w_f, int stride,
                             cudaStream_t stream, const char** err);

extern "C" int im2win_conv_basic_f32(const float* windows, const float* flt, float* out, int64_t n, int64_t c_in,
                                     int64_t c_out, int64_t h_out, int64_t w_out, int64_t row_len, int32_t h_f,
                                     int32_t w_f, int32_t stride, void* stream) {
  g_last_error[0] = '\0';
  if (!windows || !flt || !out) return fail(1, "im2win_conv_basic_f32: null pointer");
  if (n < 1 || c_in < 1 || c_out < 1 || h_out < 1 || w_out < 1 || h_f < 1 || w_f < 1 || stride < 1)
    return fail(1, "im2win_conv_basic_f32: extents must be positive");
  if (row_len != h_f * ((w_out - 1) * stride + w_f)) return fail(1, "im2win_conv_basic_f32: row_len != h_f * w_eff");
  if (int rc = bind_device_of(out)) return rc;
  const char* err = nullptr;
  int rc = im2win_launch_conv_basic(windows, flt, out, n, c_in, c_out, h_out, w_out, row_len, h_f, w_f, stride,
                                    static_cast<cudaStream_t>(stream), &err);
  return rc ? fail(rc, err) : 0;
}

// ---- direct tensor-core path for few-channel inputs (conv_tc_direct.cu) ----
int im2win_conv_direct_applies(int64_t n, int64_t c_in, int64_t h, int64_t w, int64_t c_out, int h_f, int w_f,
                               int stride, int pad, int bf16);
size_t im2win_conv_direct_workspace_bytes(int64_t c_in, int64_t c_out, int h_f, int w_f, int bf16);
int im2win_launch_conv_tc_direct(const float* x, const float* flt, float* out, void* workspace, size_t ws_bytes,
                                 int64_t n, int64_t c_in, int64_t h, int64_t w, int64_t c_out, int h_f, int w_f,
                                 int stride, int pad, int bf16, cudaStream_t stream, const char** err);

extern "C" {

int32_t im2win_conv_direct_supported(int64_t n, int64_t c_in, int64_t h, int64_t w, int64_t c_out, int32_t h_f,
                                     int32_t w_f, int32_t stride, int32_t pad, int32_t variant) {
  if (variant != IM2WIN_TF32 && variant != IM2WIN_BF16) return 0;
  if (n < 1 || c_in < 1 || h < 1 || w < 1 || c_out < 1 || h_f < 1 || w_f < 1 || stride < 1) return 0;
  return im2win_conv_direct_applies(n, c_in, h, w, c_out, h_f, w_f, stride, pad, variant == IM2WIN_BF16);
}

// The library's automatic choice between the direct kernel and channels-last copy + fused
// kernel (used by conv_im2win_opt(tc_path="auto"), CapturedConv and the host pipeline).
// Measured on B200 (tools/tc_kernels.py, N=128, copy + conv): direct wins for BF16 when the
// fused kernel's window boxes are short -- several output rows per tile (w_out <= 64: 11x11
// stride-4 layers) or a tiny window (K <= 32) -- and loses elsewhere (7x7 stride 2; TF32).
int32_t im2win_conv_direct_preferred(int64_t n, int64_t c_in, int64_t h, int64_t w, int64_t c_out, int32_t h_f,
                                     int32_t w_f, int32_t stride, int32_t pad, int32_t variant) {
  if (variant != IM2WIN_BF16 && variant != IM2WIN_TF32) return 0;
  if (!im2win_conv_direct_supported(n, c_in, h, w, c_out, h_f, w_f, stride, pad, variant)) return 0;
  // measured (bench.py, N=128, copy + conv vs direct): conv1/conv2 (Wo 55-56) BF16 166-173 TF direct vs
  // 116-120 through the channels-last copy, TF32 111-116 vs 97-103; wide outputs (conv3, conv7) are
  // faster through the copy
  const int64_t w_out = (w + 2 * pad - w_f) / stride + 1;
  return w_out <= 64 ? 1 : 0;
}

size_t im2win_conv_direct_workspace(int64_t c_in, int64_t c_out, int32_t h_f, int32_t w_f, int32_t variant) {
  return im2win_conv_direct_workspace_bytes(c_in, c_out, h_f, w_f, variant == IM2WIN_BF16);
}

int im2win_conv_direct(const float* x, const float* flt, float* out, int64_t n, int64_t c_in, int64_t h, int64_t w,
                       int64_t c_out, int32_t h_f, int32_t w_f, int32_t stride, int32_t pad, int32_t variant,
                       void* workspace, size_t workspace_bytes, void* stream) {
  g_last_error[0] = '\0';
  if (!x || !flt || !out || !workspace) return fail(1, "im2win_conv_direct: null pointer");
  if (variant != IM2WIN_TF32 && variant != IM2WIN_BF16)
    return fail(1, "im2win_conv_direct: variant must be IM2WIN_TF32 or IM2WIN_BF16");
  if (n < 1 || c_in < 1 || h < 1 || w < 1 || c_out < 1 || h_f < 1 || w_f < 1 || stride < 1 || pad < 0)
    return fail(1, "im2win_conv_direct: extents must be positive");
  if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0) return fail(1, "im2win_conv_direct: workspace alignment");
  if (int rc = bind_device_of(out)) return rc;
  const char* err = nullptr;
  int rc = im2win_launch_conv_tc_direct(x, flt, out, workspace, workspace_bytes, n, c_in, h, w, c_out, h_f, w_f,
                                        stride, pad, variant == IM2WIN_BF16, static_cast<cudaStream_t>(stream), &err);
  return rc ? fail(rc, err) : 0;
}

}  // extern "C"
