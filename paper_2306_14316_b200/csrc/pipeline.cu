// Host-buffer entry point: the whole reference call (numpy in -> numpy out,
// winconv conv_im2win_opt, /root/reference/pkg/src/winconv/kernels/optimized.py:237-241)
// with the host<->device copies overlapped against the kernels.
//
// Images are independent (reference.py:78-90), so the batch is cut into chunks
// of `chunk` images (default n/4) and run as a three-stream software pipeline per device:
//
//   h2d  : copy input chunk k            -> in[k%2]        (waits xf[k-2])
//   comp : transform in[k%2] -> Ĩ,  conv Ĩ -> out[k%2]      (waits h2d[k], d2h[k-2])
//   d2h  : copy out[k%2]                  -> host output   (waits conv[k])
//
// so PCIe upload, compute and PCIe download of consecutive chunks run at the
// same time (two copy engines + the SMs).  The per-chunk kernels are the same
// C-ABI entry points a device caller uses (im2win_transform_f32 +
// im2win_conv_f32 for the FP32 variants; im2win_nchw_to_nhwc +
// im2win_conv_fused for TF32/BF16), so results are bit-identical to the
// device path.  Host buffers should be page-locked for the copies to overlap;
// pageable buffers work but serialise.  The call blocks until the output is
// on the host.  The caller provides the device workspace
// (im2win_conv_host_workspace_bytes); the library allocates nothing.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/im2win_sm100.h"

// capi.cu: stores the message returned by im2win_last_error()
int im2win_set_error(int code, const char* msg);

namespace {

constexpr int kMaxDev = 64;
constexpr int kMaxDepth = 8;  // input / output chunk buffers in flight (runtime depth <= this)
constexpr int kRing = 256;  // completion events of non-blocking submissions

struct DevPipe {
  bool ready = false;
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  cudaEvent_t start = nullptr;
  cudaEvent_t in_ready[kMaxDepth], xf_done[kMaxDepth], conv_done[kMaxDepth], out_done[kMaxDepth];
  cudaEvent_t done[kRing];
  int64_t submitted = 0;  // tickets issued on this device (ticket t -> done[t % kRing])
  std::mutex mu;
};

DevPipe g_pipes[kMaxDev];

struct Geometry {
  int64_t n, c_in, h, w, c_out, h_out, w_out, w_eff;
  int h_f, w_f, stride, pad;
  bool tc, direct;  // direct: the few-channel TC kernel reads the NCHW chunk itself
  int64_t pitch;  // channels-last pitch for the TC path
  size_t in_elems, mid_bytes, out_elems, flt_elems, conv_ws;
};

size_t align_up(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

// FP32 chunks: windows gathered straight from NCHW (default) or via Ĩ (IM2WIN_FP32_PATH=windows),
// the same rule as kernels.nchw_direct
bool fp32_nchw_path() {
  const char* e = getenv("IM2WIN_FP32_PATH");
  return !(e && std::strcmp(e, "windows") == 0);
}

Geometry geometry(int64_t n_chunk, int64_t c_in, int64_t h, int64_t w, int64_t c_out, int h_f, int w_f, int stride,
                  int pad, int variant) {
  Geometry g{};
  g.n = n_chunk;
  g.c_in = c_in;
  g.h = h;
  g.w = w;
  g.c_out = c_out;
  g.h_f = h_f;
  g.w_f = w_f;
  g.stride = stride;
  g.pad = pad;
  g.h_out = (h + 2 * pad - h_f) / stride + 1;
  g.w_out = (w + 2 * pad - w_f) / stride + 1;
  g.w_eff = (g.w_out - 1) * stride + w_f;
  g.tc = variant == IM2WIN_TF32 || variant == IM2WIN_BF16;
  const int q = variant == IM2WIN_BF16 ? 8 : 4;
  g.pitch = (c_in + q - 1) / q * q;
  g.in_elems = static_cast<size_t>(n_chunk * c_in * h * w);
  g.out_elems = static_cast<size_t>(n_chunk * c_out * g.h_out * g.w_out);
  g.flt_elems = static_cast<size_t>(c_out * c_in * h_f * w_f);
  g.direct = g.tc && im2win_conv_direct_preferred(n_chunk, c_in, h, w, c_out, h_f, w_f, stride, pad, variant);
  if (g.direct) {
    g.mid_bytes = 0;
    g.conv_ws = im2win_conv_direct_workspace(c_in, c_out, h_f, w_f, variant);
  } else if (g.tc) {
    g.mid_bytes = static_cast<size_t>(n_chunk * (h + 2 * pad) * (w + 2 * pad) * g.pitch) * (variant == IM2WIN_BF16 ? 2 : 4);
    // unpadded: the one-call fused entry (channels-last copy inside the conv kernel or just before it)
    g.conv_ws = pad == 0 ? im2win_conv_fused_nchw_workspace_bytes(n_chunk, c_in, c_out, h_f, w_f)
                         : im2win_conv_fused_workspace_bytes(c_in, c_out, h_f, w_f);
  } else {
    g.mid_bytes = static_cast<size_t>(n_chunk * c_in * g.h_out * h_f * g.w_eff) * 4;
    g.conv_ws = im2win_conv_workspace_bytes(c_in, c_out, h_f, w_f, variant);
  }
  return g;
}

// Chunk buffers per call: one per chunk up to kMaxDepth, so a call's compute never waits
// for its own downloads (measured: with 2 buffers, compute of a download-heavy layer is
// paced by PCIe and stalls every later call on the compute stream).  IM2WIN_HOST_DEPTH caps it.
int depth_for(int64_t n_chunks) {
  static int cap = [] {
    const char* e = getenv("IM2WIN_HOST_DEPTH");
    int v = e ? atoi(e) : kMaxDepth;
    return v < 1 ? 1 : (v > kMaxDepth ? kMaxDepth : v);
  }();
  return static_cast<int>(std::min<int64_t>(n_chunks, cap));
}

size_t workspace_bytes(const Geometry& g, int64_t n_chunks) {
  return align_up(g.flt_elems * 4) + align_up(g.conv_ws) + align_up(g.mid_bytes) +
         depth_for(n_chunks) * (align_up(g.in_elems * 4) + align_up(g.out_elems * 4));
}

int64_t pick_chunk(int64_t n, int64_t chunk) {
  if (chunk > 0) return std::min(chunk, n);
  // 4 chunks per call (measured best over 4..32 images per chunk at N=128, tools/e2e_sweep.py):
  // larger chunks keep the kernels efficient; consecutive non-blocking calls overlap the fill/drain
  return std::max<int64_t>(1, (n + 3) / 4);
}

// Restores the calling thread's current device on scope exit: the host entry points bind
// the workspace's device, and the caller's later default-device work must not move with it.
struct DeviceGuard {
  int saved = -1;
  DeviceGuard() {
    if (cudaGetDevice(&saved) != cudaSuccess) saved = -1;
  }
  ~DeviceGuard() {
    if (saved >= 0) cudaSetDevice(saved);
  }
};

}  // namespace

extern "C" {

size_t im2win_conv_host_workspace_bytes(int64_t n, int64_t c_in, int64_t h, int64_t w, int64_t c_out, int32_t h_f,
                                        int32_t w_f, int32_t stride, int32_t pad, int32_t variant,
                                        int64_t chunk_images) {
  if (n < 1 || c_in < 1 || h < 1 || w < 1 || c_out < 1 || h_f < 1 || w_f < 1 || stride < 1 || pad < 0 ||
      h_f > h + 2 * pad || w_f > w + 2 * pad)
    return 0;
  const int64_t cn = pick_chunk(n, chunk_images);
  return workspace_bytes(geometry(cn, c_in, h, w, c_out, h_f, w_f, stride, pad, variant), (n + cn - 1) / cn);
}

}  // extern "C"

static int host_conv(const float* host_in, const float* host_flt, float* host_out, int64_t n, int64_t c_in,
                     int64_t h, int64_t w, int64_t c_out, int32_t h_f, int32_t w_f, int32_t stride, int32_t pad,
                     const im2win_tile_plan* plan, int32_t variant, int64_t chunk_images, void* workspace,
                     size_t ws_bytes, void* stream, int64_t* ticket) {
  if (!host_in || !host_flt || !host_out || !workspace) return im2win_set_error(1, "im2win_conv_host_f32: null pointer");
  if (n < 1 || c_in < 1 || h < 1 || w < 1 || c_out < 1 || h_f < 1 || w_f < 1 || stride < 1 || pad < 0)
    return im2win_set_error(1, "im2win_conv_host_f32: extents must be positive");
  if (h_f > h + 2 * pad || w_f > w + 2 * pad)
    return im2win_set_error(1, "im2win_conv_host_f32: filter larger than input");
  if (variant < IM2WIN_FP32_EXACT || variant > IM2WIN_BF16)
    return im2win_set_error(1, "im2win_conv_host_f32: unknown variant");
  const int64_t cn = pick_chunk(n, chunk_images);
  const Geometry g = geometry(cn, c_in, h, w, c_out, h_f, w_f, stride, pad, variant);
  const int64_t n_chunks = (n + cn - 1) / cn;
  if (ws_bytes < workspace_bytes(g, n_chunks)) return im2win_set_error(1, "im2win_conv_host_f32: workspace too small");

  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, workspace) != cudaSuccess || attr.type != cudaMemoryTypeDevice)
    return im2win_set_error(1, "im2win_conv_host_f32: workspace is not device memory");
  const int dev = attr.device;
  if (dev < 0 || dev >= kMaxDev) return im2win_set_error(1, "im2win_conv_host_f32: device index out of range");
  DeviceGuard guard;
  cudaSetDevice(dev);
  DevPipe& P = g_pipes[dev];
  std::lock_guard<std::mutex> lock(P.mu);
  if (!P.ready) {
    cudaStreamCreateWithFlags(&P.h2d, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&P.comp, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&P.d2h, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&P.start, cudaEventDisableTiming);
    for (int i = 0; i < kMaxDepth; ++i) {
      cudaEventCreateWithFlags(&P.in_ready[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&P.xf_done[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&P.conv_done[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&P.out_done[i], cudaEventDisableTiming);
    }
    for (int i = 0; i < kRing; ++i) cudaEventCreateWithFlags(&P.done[i], cudaEventDisableTiming);
    if (cudaGetLastError() != cudaSuccess) return im2win_set_error(2, "im2win_conv_host_f32: stream setup failed");
    P.ready = true;
  }

  // carve the workspace
  char* base = static_cast<char*>(workspace);
  float* d_flt = reinterpret_cast<float*>(base);
  base += align_up(g.flt_elems * 4);
  void* conv_ws = base;
  base += align_up(g.conv_ws);
  void* mid = base;
  base += align_up(g.mid_bytes);
  const int D = depth_for(n_chunks);
  float* d_in[kMaxDepth];
  float* d_out[kMaxDepth];
  for (int i = 0; i < D; ++i) {
    d_in[i] = reinterpret_cast<float*>(base);
    base += align_up(g.in_elems * 4);
    d_out[i] = reinterpret_cast<float*>(base);
    base += align_up(g.out_elems * 4);
  }

  // everything is ordered after the caller's prior work on `stream` (it may own the workspace)
  cudaStream_t user = static_cast<cudaStream_t>(stream);
  cudaEventRecord(P.start, user);
  cudaStreamWaitEvent(P.h2d, P.start, 0);
  cudaStreamWaitEvent(P.comp, P.start, 0);
  cudaStreamWaitEvent(P.d2h, P.start, 0);
  cudaMemcpyAsync(d_flt, host_flt, g.flt_elems * 4, cudaMemcpyHostToDevice, P.h2d);  // before chunk 0's in_ready

  const int64_t img_in = c_in * h * w;
  const int64_t img_out = c_out * g.h_out * g.w_out;
  int rc = 0;
  for (int64_t k = 0; k < n_chunks && rc == 0; ++k) {
    const int s = static_cast<int>(k % D);
    const int64_t i0 = k * cn;
    const int64_t nk = std::min(cn, n - i0);
    // upload (buffer s was last read by chunk k-2's transform)
    if (k >= D) cudaStreamWaitEvent(P.h2d, P.xf_done[s], 0);
    cudaMemcpyAsync(d_in[s], host_in + i0 * img_in, static_cast<size_t>(nk * img_in) * 4, cudaMemcpyHostToDevice,
                    P.h2d);
    cudaEventRecord(P.in_ready[s], P.h2d);
    // compute (output buffer s was last read by chunk k-2's download)
    cudaStreamWaitEvent(P.comp, P.in_ready[s], 0);
    if (k >= D) cudaStreamWaitEvent(P.comp, P.out_done[s], 0);
    if (g.direct) {
      // the direct kernel reads the chunk's NCHW input itself: buffer s is free once it finishes
      rc = im2win_conv_direct(d_in[s], d_flt, d_out[s], nk, c_in, h, w, c_out, h_f, w_f, stride, pad, variant,
                              conv_ws, g.conv_ws, P.comp);
      cudaEventRecord(P.xf_done[s], P.comp);
    } else if (g.tc && pad == 0) {
      // reads the chunk's NCHW input until the conv finishes: buffer s is free after it
      rc = im2win_conv_fused_nchw(d_in[s], mid, d_flt, d_out[s], nk, c_in, h, w, c_out, h_f, w_f, stride, variant,
                                  conv_ws, g.conv_ws, P.comp);
      cudaEventRecord(P.xf_done[s], P.comp);
    } else if (g.tc) {
      rc = im2win_nchw_to_nhwc_padded(d_in[s], mid, nk, c_in, h, w, variant == IM2WIN_BF16 ? 1 : 0, pad, P.comp);
      cudaEventRecord(P.xf_done[s], P.comp);
      if (!rc)
        rc = im2win_conv_fused(mid, d_flt, d_out[s], nk, c_in, h + 2 * pad, w + 2 * pad, c_out, h_f, w_f, stride,
                               variant, conv_ws, g.conv_ws, P.comp);
    } else if (pad == 0 && (!plan || plan->micro_kernel) && fp32_nchw_path()) {
      // the tiled kernel gathers the windows from the chunk's NCHW input (no Ĩ; same bits):
      // input buffer s is free once the conv finishes
      rc = im2win_conv_nchw_f32(d_in[s], d_flt, d_out[s], nk, c_in, h, w, c_out, h_f, w_f, stride, plan, variant,
                                conv_ws, g.conv_ws, P.comp);
      cudaEventRecord(P.xf_done[s], P.comp);
    } else {
      rc = im2win_transform_f32_padded(d_in[s], static_cast<float*>(mid), nk, c_in, h, w, h_f, w_f, stride, pad,
                                       P.comp);
      cudaEventRecord(P.xf_done[s], P.comp);
      if (!rc)
        rc = im2win_conv_f32(static_cast<float*>(mid), d_flt, d_out[s], nk, c_in, c_out, g.h_out, g.w_out,
                             static_cast<int64_t>(h_f) * g.w_eff, h_f, w_f, stride, plan, variant, conv_ws, g.conv_ws,
                             P.comp);
    }
    cudaEventRecord(P.conv_done[s], P.comp);
    // download
    cudaStreamWaitEvent(P.d2h, P.conv_done[s], 0);
    cudaMemcpyAsync(host_out + i0 * img_out, d_out[s], static_cast<size_t>(nk * img_out) * 4,
                    cudaMemcpyDeviceToHost, P.d2h);
    cudaEventRecord(P.out_done[s], P.d2h);
  }
  if (rc) {
    // an entry point failed mid-loop: chunks already queued may still be reading or writing
    // the workspace; drain all three streams so the caller can free or reuse it at once
    cudaStreamSynchronize(P.h2d);
    cudaStreamSynchronize(P.comp);
    cudaStreamSynchronize(P.d2h);
  }
  if (ticket) {
    // non-blocking: completion is ticket-tracked; the caller's stream is not made to wait,
    // so the next submission's uploads overlap this one's downloads
    const int64_t t = P.submitted++;
    cudaEventRecord(P.done[t % kRing], P.d2h);
    *ticket = (static_cast<int64_t>(dev) << 48) | t;
    if (rc) return rc;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : im2win_set_error(2, cudaGetErrorString(e));
  }
  // blocking: the caller's stream resumes after the last download; the call itself blocks on it
  cudaEventRecord(P.start, P.d2h);
  cudaStreamWaitEvent(user, P.start, 0);
  cudaError_t e = cudaStreamSynchronize(P.d2h);
  if (rc) return rc;  // message already set by the failing entry point
  if (e != cudaSuccess) return im2win_set_error(2, cudaGetErrorString(e));
  e = cudaGetLastError();
  if (e != cudaSuccess) return im2win_set_error(2, cudaGetErrorString(e));
  return 0;
}

extern "C" {

int im2win_conv_host_f32(const float* host_in, const float* host_flt, float* host_out, int64_t n, int64_t c_in,
                         int64_t h, int64_t w, int64_t c_out, int32_t h_f, int32_t w_f, int32_t stride, int32_t pad,
                         const im2win_tile_plan* plan, int32_t variant, int64_t chunk_images, void* workspace,
                         size_t ws_bytes, void* stream) {
  return host_conv(host_in, host_flt, host_out, n, c_in, h, w, c_out, h_f, w_f, stride, pad, plan, variant,
                   chunk_images, workspace, ws_bytes, stream, nullptr);
}

int im2win_conv_host_submit(const float* host_in, const float* host_flt, float* host_out, int64_t n, int64_t c_in,
                            int64_t h, int64_t w, int64_t c_out, int32_t h_f, int32_t w_f, int32_t stride, int32_t pad,
                            const im2win_tile_plan* plan, int32_t variant, int64_t chunk_images, void* workspace,
                            size_t ws_bytes, void* stream, int64_t* ticket) {
  if (!ticket) return im2win_set_error(1, "im2win_conv_host_submit: null ticket");
  return host_conv(host_in, host_flt, host_out, n, c_in, h, w, c_out, h_f, w_f, stride, pad, plan, variant,
                   chunk_images, workspace, ws_bytes, stream, ticket);
}

int im2win_conv_host_wait(int64_t ticket) {
  const int dev = static_cast<int>(ticket >> 48);
  const int64_t t = ticket & ((static_cast<int64_t>(1) << 48) - 1);
  if (dev < 0 || dev >= kMaxDev) return im2win_set_error(1, "im2win_conv_host_wait: bad ticket");
  DevPipe& P = g_pipes[dev];
  cudaEvent_t ev;
  {
    std::lock_guard<std::mutex> lock(P.mu);
    if (!P.ready || t >= P.submitted) return im2win_set_error(1, "im2win_conv_host_wait: bad ticket");
    // the d2h stream is in order: if slot t was re-recorded by a later ticket, that one
    // completes after t, so waiting on it is still correct (just later)
    ev = P.done[t % kRing];
  }
  DeviceGuard guard;
  cudaSetDevice(dev);
  cudaError_t e = cudaEventSynchronize(ev);
  return e == cudaSuccess ? 0 : im2win_set_error(2, cudaGetErrorString(e));
}

}  // extern "C"
