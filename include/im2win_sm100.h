/*
 * im2win_sm100.h — C ABI of libim2win_sm100.so, the B200 (sm_100a) im2win
 * transform and im2win convolution.
 *
 * The reference (`winconv`, pure Python + numba) has no C ABI: its native
 * seam is two numba kernels that already follow the "caller allocates, flat
 * buffers + integer scalars, no return value" convention.  Each entry point
 * below replaces one of them one-for-one:
 *
 *   im2win_transform_f32   <- _im2win_fill(src, dst, h_f, w_eff, stride)
 *                             /root/reference/pkg/src/winconv/layouts.py:73-83,
 *                             called from im2win() at layouts.py:94
 *   im2win_conv_f32        <- _tiled_kernel(windows_flat, flt_flat, out_flat,
 *                             dim_m, dim_n, dim_k, c_in, c_out, h_out, w_out,
 *                             row_len, h_f, w_f, stride, m_b, n_b, k_b, m_t,
 *                             n_t, use_vec, use_pf)
 *                             kernels/optimized.py:66-214, called from
 *                             compute_from_windows_opt() at optimized.py:228-233
 *
 * Conventions (same as the reference seam):
 *   - every pointer is device memory on the current CUDA device; the caller
 *     allocates all outputs and the optional workspace (layouts.py:93,
 *     optimized.py:226); the library never allocates device memory;
 *   - tensors are float32, C-contiguous, NCHW (tensors.py:1-6);
 *   - validation of shapes/geometry happens in the host layer before the
 *     call (ShapeError / GeometryError / PlanError, errors.py:4-33); the
 *     library re-checks index ranges and returns nonzero on violation;
 *   - work is enqueued on `stream` (a cudaStream_t; NULL = legacy default
 *     stream) and the call returns without synchronising;
 *   - return 0 on success; nonzero = error, message via im2win_last_error().
 */
#ifndef IM2WIN_SM100_H
#define IM2WIN_SM100_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Arithmetic variants of the convolution. */
enum im2win_variant {
  IM2WIN_FP32_EXACT = 0, /* FMUL+FADD, ascending k: bit-exact with the reference */
  IM2WIN_FP32_FMA = 1,   /* FFMA, ascending k: within 1e-4 of the reference        */
  IM2WIN_TF32 = 2,       /* tcgen05 kind::tf32, fp32 accumulate in TMEM            */
  IM2WIN_BF16 = 3        /* tcgen05 kind::f16 (bf16 operands), fp32 accumulate     */
};

/* GPU tile plan; mirrors winconv TilePlan (kernels/plan.py:11-48).
 * block_cfg < 0 lets the library pick the tile for the shape. */
typedef struct im2win_tile_plan {
  int32_t block_cfg;              /* index of a compiled CTA tile, or -1        */
  int32_t micro_kernel;           /* 1: 8x8 register micro-tile; 0: 1x1         */
  int32_t vectorized_load;        /* 1: 128-bit shared-memory fragment loads     */
  int32_t prefetch_double_buffer; /* 1: multi-stage async prefetch ring          */
} im2win_tile_plan;

/* Window-order transform (layouts.py:73-95).
 * src: (n, c, h, w) float32; dst: (n, c, h_out, h_f * w_eff) float32 where
 * h_out = (h - h_f) / stride + 1, w_eff = (w_out - 1) * stride + w_f.
 * Bit-exact copy: dst[i,r,m,col*h_f+u] = src[i,r,m*stride+u,col].
 * Any 4-byte aligned src/dst (numpy/torch views at an element offset included); 16-byte
 * aligned buffers take the TMA bulk-copy kernel. */
int im2win_transform_f32(const float* src, float* dst, int64_t n, int64_t c, int64_t h,
                         int64_t w, int32_t h_f, int32_t w_f, int32_t stride, void* stream);

/* Extension: the same transform of the input zero-padded by `pad` on every side
 * (the reference has no padding; callers pre-pad).  The padded input is never
 * materialised: dst is (n, c, h_out, h_f * w_eff) for the padded geometry
 * h_out = (h + 2*pad - h_f) / stride + 1, w_eff = (w_out - 1) * stride + w_f,
 * bit-identical to im2win_transform_f32 of the explicitly padded input.
 * src and dst must be 16-byte aligned when pad > 0. */
int im2win_transform_f32_padded(const float* src, float* dst, int64_t n, int64_t c, int64_t h,
                                int64_t w, int32_t h_f, int32_t w_f, int32_t stride, int32_t pad,
                                void* stream);

/* Bytes of device workspace im2win_conv_f32 needs (packed filter + offsets); the
 * workspace must be 16-byte aligned. */
size_t im2win_conv_workspace_bytes(int64_t c_in, int64_t c_out, int32_t h_f, int32_t w_f,
                                   int32_t variant);

/* im2win convolution on an already-transformed input (optimized.py:217-234).
 * windows: (n, c_in, h_out, row_len) from im2win_transform_f32;
 * flt: (c_out, c_in, h_f, w_f); out: (n, c_out, h_out, w_out).
 * plan may be NULL (library default). */
int im2win_conv_f32(const float* windows, const float* flt, float* out, int64_t n, int64_t c_in,
                    int64_t c_out, int64_t h_out, int64_t w_out, int64_t row_len, int32_t h_f,
                    int32_t w_f, int32_t stride, const im2win_tile_plan* plan, int32_t variant,
                    void* workspace, size_t workspace_bytes, void* stream);

/* The FP32 conv_im2win_opt without a materialised Ĩ (replaces the transform + _tiled_kernel
 * pair of pkg/src/winconv/kernels/optimized.py:237-241 in one launch): the same kernels gather
 * every window element Ĩ[img][c][oh][(ow*s + fw)*Hf + fh] = x[img][c][oh*s + fh][ow*s + fw]
 * straight from the NCHW input x (n, c_in, h, w), in the reference's k order -- bit-identical
 * to im2win_transform_f32 + im2win_conv_f32.  variant = IM2WIN_FP32_EXACT or IM2WIN_FP32_FMA;
 * plan as for im2win_conv_f32 (micro_kernel must be 1); workspace as im2win_conv_workspace_bytes. */
int im2win_conv_nchw_f32(const float* x, const float* flt, float* out, int64_t n, int64_t c_in,
                         int64_t h, int64_t w, int64_t c_out, int32_t h_f, int32_t w_f, int32_t stride,
                         const im2win_tile_plan* plan, int32_t variant, void* workspace,
                         size_t workspace_bytes, void* stream);

/* Paper Alg. 2 basic kernel: one output per thread, operands from global memory
 * (replaces _basic_window_kernel, kernels/reference.py:180-206, called at :215).
 * Bit-exact like im2win_conv_f32 with IM2WIN_FP32_EXACT. */
int im2win_conv_basic_f32(const float* windows, const float* flt, float* out, int64_t n,
                          int64_t c_in, int64_t c_out, int64_t h_out, int64_t w_out,
                          int64_t row_len, int32_t h_f, int32_t w_f, int32_t stride, void* stream);

/* ---- Tensor-core fast path (extension; no counterpart in the reference) ----
 * The channels-innermost form of the window layout, Ĩcl[n*Ho+oh][col][fh][c] =
 * X[n][c][oh*stride+fh][col] (col < w_eff), makes every pixel's window one
 * contiguous run of c_in*h_f*w_f elements, so the tcgen05 kernel streams window
 * tiles with TMA and no gather.  dtype 0 stores float32 (TF32 variant), 1 bf16.
 * Requires c_in * element size to be a multiple of 16 bytes for im2win_conv_cl. */
int im2win_transform_cl(const float* src, void* dst, int64_t n, int64_t c, int64_t h, int64_t w,
                        int32_t h_f, int32_t w_f, int32_t stride, int32_t dtype, void* stream);

size_t im2win_conv_cl_workspace_bytes(int64_t c_in, int64_t c_out, int32_t h_f, int32_t w_f);

/* variant = IM2WIN_TF32 (windows_cl float32) or IM2WIN_BF16 (windows_cl bf16). */
int im2win_conv_cl(const void* windows_cl, const float* flt, float* out, int64_t n, int64_t c_in,
                   int64_t c_out, int64_t h_out, int64_t w_out, int32_t h_f, int32_t w_f,
                   int32_t stride, int32_t variant, void* workspace, size_t workspace_bytes,
                   void* stream);

/* ---- Fused tensor-core path (extension): no materialised window tensor ----
 * im2win_nchw_to_nhwc copies X to channels-last (dtype 0 f32, 1 bf16; c % 4 == 0);
 * im2win_conv_fused then reads every window row Xnhwc[n][oh*s+fh][ow*s..ow*s+w_f-1][:]
 * with one 5-D TMA box per K-slab (the windows are built by the TMA engine). */
int im2win_nchw_to_nhwc(const float* src, void* dst, int64_t n, int64_t c, int64_t h, int64_t w,
                        int32_t dtype, void* stream);

/* The same copy into a spatially zero-padded destination (n, h + 2*pad, w + 2*pad,
 * pitch): border pixels are written as zeros, so im2win_conv_fused on it with the
 * padded extents computes the padded convolution. */
int im2win_nchw_to_nhwc_padded(const float* src, void* dst, int64_t n, int64_t c, int64_t h, int64_t w,
                               int32_t dtype, int32_t pad, void* stream);

size_t im2win_conv_fused_workspace_bytes(int64_t c_in, int64_t c_out, int32_t h_f, int32_t w_f);

int im2win_conv_fused(const void* x_nhwc, const float* flt, float* out, int64_t n, int64_t c_in,
                      int64_t h, int64_t w, int64_t c_out, int32_t h_f, int32_t w_f, int32_t stride,
                      int32_t variant, void* workspace, size_t workspace_bytes, void* stream);

/* One call for the whole TF32/BF16 conv_im2win_opt (replaces the numba conv_im2win_opt,
 * pkg/src/winconv/kernels/optimized.py:237-241, for the tensor-core variants): x is the
 * NCHW float32 input; x_nhwc is caller-provided scratch of n*h*w*pitch elements
 * (pitch = channel pitch of im2win_nchw_to_nhwc for the variant's dtype) that extra warps
 * of the conv kernel fill while the tensor cores run, instead of a separate copy kernel
 * before it.  Same results as im2win_nchw_to_nhwc + im2win_conv_fused, bit for bit. */
size_t im2win_conv_fused_nchw_workspace_bytes(int64_t n, int64_t c_in, int64_t c_out, int32_t h_f,
                                              int32_t w_f);

int im2win_conv_fused_nchw(const float* x, void* x_nhwc, const float* flt, float* out, int64_t n,
                           int64_t c_in, int64_t h, int64_t w, int64_t c_out, int32_t h_f, int32_t w_f,
                           int32_t stride, int32_t variant, void* workspace, size_t workspace_bytes,
                           void* stream);

/* ---- Direct tensor-core path for few-channel inputs (extension) ----
 * For C <= 16 (the RGB input layers) producer warps build each output pixel's im2win
 * window (k = (c, fh, fw), C*Hf*Wf values) from an input patch staged in shared memory
 * and feed tcgen05 directly: no channels-last copy, no TMA window boxes.  x is the NCHW
 * float32 input; pad zero-pads it on every side.  variant = IM2WIN_TF32 or IM2WIN_BF16.
 * im2win_conv_direct_supported returns 1 when the shape fits (else use the fused path). */
int32_t im2win_conv_direct_supported(int64_t n, int64_t c_in, int64_t h, int64_t w, int64_t c_out,
                                     int32_t h_f, int32_t w_f, int32_t stride, int32_t pad, int32_t variant);

/* 1 when the library's automatic path would pick the direct kernel over copy + fused. */
int32_t im2win_conv_direct_preferred(int64_t n, int64_t c_in, int64_t h, int64_t w, int64_t c_out,
                                     int32_t h_f, int32_t w_f, int32_t stride, int32_t pad, int32_t variant);

size_t im2win_conv_direct_workspace(int64_t c_in, int64_t c_out, int32_t h_f, int32_t w_f, int32_t variant);

int im2win_conv_direct(const float* x, const float* flt, float* out, int64_t n, int64_t c_in, int64_t h,
                       int64_t w, int64_t c_out, int32_t h_f, int32_t w_f, int32_t stride, int32_t pad,
                       int32_t variant, void* workspace, size_t workspace_bytes, void* stream);

/* ---- Host-buffer entry point (extension of conv_im2win_opt, optimized.py:237-241) ----
 * The reference is called with host (numpy) operands and returns a host array.
 * This runs transform + conv over host buffers: the batch is cut into chunks of
 * chunk_images (<= 0: about n/8) and a three-stream pipeline overlaps the
 * upload of chunk k+1, the kernels of chunk k and the download of chunk k-1.
 * host_in (n,c_in,h,w), host_flt (c_out,c_in,h_f,w_f), host_out (n,c_out,h_out,w_out);
 * pad >= 0 zero-pads the input on every side (0 = the reference's unpadded conv)
 * are host memory (page-locked for overlap); workspace is device memory of at
 * least im2win_conv_host_workspace_bytes(...) bytes on the device to run on.
 * Ordered after prior work on `stream`; blocks until host_out is written.
 * Results are bit-identical to im2win_transform_f32 + im2win_conv_f32
 * (FP32 variants) or im2win_nchw_to_nhwc + im2win_conv_fused (TF32/BF16). */
size_t im2win_conv_host_workspace_bytes(int64_t n, int64_t c_in, int64_t h, int64_t w, int64_t c_out,
                                        int32_t h_f, int32_t w_f, int32_t stride, int32_t pad,
                                        int32_t variant, int64_t chunk_images);

int im2win_conv_host_f32(const float* host_in, const float* host_flt, float* host_out, int64_t n,
                         int64_t c_in, int64_t h, int64_t w, int64_t c_out, int32_t h_f, int32_t w_f,
                         int32_t stride, int32_t pad, const im2win_tile_plan* plan, int32_t variant,
                         int64_t chunk_images, void* workspace, size_t workspace_bytes, void* stream);

/* Non-blocking form: enqueues the same work and returns at once with a ticket;
 * host_out (and the workspace, which must stay allocated and unused by others)
 * are valid/free after im2win_conv_host_wait(ticket) returns 0.  Consecutive
 * submissions on one device overlap (uploads of one with downloads of the
 * previous).  The caller's stream is only used to order the start. */
int im2win_conv_host_submit(const float* host_in, const float* host_flt, float* host_out, int64_t n,
                            int64_t c_in, int64_t h, int64_t w, int64_t c_out, int32_t h_f, int32_t w_f,
                            int32_t stride, int32_t pad, const im2win_tile_plan* plan, int32_t variant,
                            int64_t chunk_images, void* workspace, size_t workspace_bytes, void* stream,
                            int64_t* ticket);

int im2win_conv_host_wait(int64_t ticket);

/* Measurement utility (bench.py only): launches `blocks` x 256 threads that each
 * retire 2*32*iters flops of independent FP32 multiply-add chains; exact != 0
 * issues FMUL+FADD (the conv's bit-exact pair), else FFMA.  Used to measure the
 * CUDA-core FP32 roofline denominator on the box (not in MEASURED_PEAKS.json). */
int im2win_bench_fp32_peak(float* sink, int32_t exact, int32_t iters, int32_t blocks, void* stream);

/* Message of the last failing call on this host thread ("" if none). */
const char* im2win_last_error(void);

/* Name of the compute kernel the last successful conv call on this host thread
 * launched (which of the tile/kernel variants the library selected). */
const char* im2win_last_kernel(void);

/* Conv kernel launches made by this library so far (all threads; a layer may take two:
 * the SIMT tail split).  bench.py counts the launches of its timed region with it. */
int64_t im2win_conv_launch_count(void);

/* ABI version of this library (major*100 + minor). */
int32_t im2win_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* IM2WIN_SM100_H */
