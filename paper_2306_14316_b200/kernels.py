"""im2win convolution entry points (drop-in for winconv.kernels.optimized).

`compute_from_windows_opt` mirrors /root/reference/pkg/src/winconv/kernels/optimized.py:217-234
and `conv_im2win_opt` mirrors :237-241.  The tiled kernel (`_tiled_kernel`,
:66-214) is the sm_100a library behind `im2win_conv_f32`.

Extra keyword `variant` (default "fp32-exact") selects the arithmetic:
  fp32-exact  FMUL+FADD, ascending k  -> bitwise equal to the reference
  fp32-fma    FFMA, ascending k       -> within 1e-4 (max_rel_diff)
  tf32, bf16  tcgen05 tensor cores    -> within the stated normalized tolerance
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib
from .errors import ShapeError
from .layouts import Im2winTensor, im2win
from .plan import GemmDims, TilePlan, to_c_plan
from .tensors import DTYPE, ConvParams, Tensor4, check_conv_operands, output_dims

_workspaces: dict[tuple, torch.Tensor] = {}


def _workspace(device: torch.device, stream: int, nbytes: int) -> torch.Tensor:
    key = (device.index, stream)
    buf = _workspaces.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8, device=device)
        _workspaces[key] = buf
    return buf


def _check_ws(ws: torch.Tensor, nbytes: int) -> torch.Tensor:
    """A caller-owned workspace (e.g. one a captured CUDA graph keeps referencing)."""
    if ws.numel() * ws.element_size() < nbytes or not ws.is_cuda:
        raise ShapeError(f"workspace of {ws.numel() * ws.element_size()} bytes, need {nbytes}")
    return ws


def _variant_code(variant: str) -> int:
    try:
        return _lib.VARIANTS[variant]
    except KeyError:
        raise ValueError(f"unknown variant {variant!r}, expected one of {tuple(_lib.VARIANTS)}") from None


def conv_windows_into(win: torch.Tensor, flt: torch.Tensor, out: torch.Tensor, params: ConvParams,
                      w_eff: int, plan: TilePlan | None = None, variant: str = "fp32-exact",
                      ws: torch.Tensor | None = None) -> None:
    """Launch the convolution into a caller-allocated output (the optimized.py:228-233 seam)."""
    n_img, c_in, h_out, row_len = (int(d) for d in win.shape)
    w_out = int(out.shape[3])
    code = _variant_code(variant)
    lib = _lib.load()
    nbytes = lib.im2win_conv_workspace_bytes(c_in, params.c_out, params.h_f, params.w_f, code)
    stream = torch.cuda.current_stream(win.device).cuda_stream
    ws = _workspace(win.device, stream, nbytes) if ws is None else _check_ws(ws, nbytes)
    cplan = to_c_plan(plan)
    with torch.cuda.device(win.device):
        rc = lib.im2win_conv_f32(
            win.data_ptr(), flt.data_ptr(), out.data_ptr(), n_img, c_in, params.c_out, h_out, w_out,
            row_len, params.h_f, params.w_f, params.stride,
            None if cplan is None else _byref(cplan), code, ws.data_ptr(), ws.numel(), stream)
    _lib.check(rc)


def conv_nchw_into(x: torch.Tensor, flt: torch.Tensor, out: torch.Tensor, params: ConvParams,
                   plan: TilePlan | None = None, variant: str = "fp32-exact",
                   ws: torch.Tensor | None = None) -> None:
    """FP32 im2win convolution straight from the NCHW input (im2win_conv_nchw_f32): the tiled
    kernel gathers each window element from x in the reference's k order, so no Ĩ is written
    and the bits equal im2win_into + conv_windows_into."""
    n_img, c_in, h_in, w_in = (int(d) for d in x.shape)
    code = _variant_code(variant)
    lib = _lib.load()
    nbytes = lib.im2win_conv_workspace_bytes(c_in, params.c_out, params.h_f, params.w_f, code)
    stream = torch.cuda.current_stream(x.device).cuda_stream
    ws = _workspace(x.device, stream, nbytes) if ws is None else _check_ws(ws, nbytes)
    cplan = to_c_plan(plan)
    with torch.cuda.device(x.device):
        rc = lib.im2win_conv_nchw_f32(x.data_ptr(), flt.data_ptr(), out.data_ptr(), n_img, c_in, h_in, w_in,
                                      params.c_out, params.h_f, params.w_f, params.stride,
                                      None if cplan is None else _byref(cplan), code, ws.data_ptr(), ws.numel(),
                                      stream)
    _lib.check(rc)


def _byref(x):
    import ctypes

    return ctypes.byref(x)


def compute_from_windows_opt(windows: Im2winTensor, flt, params: ConvParams,
                             plan: TilePlan | None = None, *, variant: str = "fp32-exact") -> Tensor4:
    """Tiled convolution on an already-transformed input (optimized.py:217-234)."""
    f = flt if isinstance(flt, Tensor4) else Tensor4(flt)
    if f.dims != params.filter_dims:
        raise ShapeError(f"filter dims {f.dims} do not match params {params.filter_dims}")
    # the reference leaves these unchecked (optimized.py:217-226); a GPU kernel must not read out of bounds
    if windows.c_in != params.c_in:
        raise ShapeError(f"windows have {windows.c_in} channels, params expect {params.c_in}")
    if (windows.h_f, windows.w_f, windows.stride) != (params.h_f, params.w_f, params.stride):
        raise ShapeError("window tensor geometry does not match params")
    fd = f.data if f.device == windows.data.device else f.data.to(windows.data.device)
    # GemmDims is computed for parity with the reference call stack (optimized.py:222-223)
    GemmDims(params.c_out, windows.n * windows.h_out * windows.w_out,
             params.c_in * params.h_f * params.w_f)
    out = torch.empty((windows.n, params.c_out, windows.h_out, windows.w_out), dtype=DTYPE,
                      device=windows.data.device)
    conv_windows_into(windows.data, fd, out, params, windows.w_eff, plan, variant)
    return Tensor4(out)


def basic_windows_into(win: torch.Tensor, flt: torch.Tensor, out: torch.Tensor, params: ConvParams) -> None:
    """Paper Alg. 2 basic kernel into a caller-allocated output (reference.py:209-219 seam)."""
    n_img, c_in, h_out, row_len = (int(d) for d in win.shape)
    w_out = int(out.shape[3])
    with torch.cuda.device(win.device):
        rc = _lib.load().im2win_conv_basic_f32(
            win.data_ptr(), flt.data_ptr(), out.data_ptr(), n_img, c_in, params.c_out, h_out, w_out, row_len,
            params.h_f, params.w_f, params.stride, torch.cuda.current_stream(win.device).cuda_stream)
    _lib.check(rc)


def compute_from_windows_basic(windows: Im2winTensor, flt, params: ConvParams) -> Tensor4:
    """Basic window-order convolution on an already-transformed input (reference.py:209-219)."""
    f = flt if isinstance(flt, Tensor4) else Tensor4(flt)
    if f.dims != params.filter_dims:
        raise ShapeError(f"filter dims {f.dims} do not match params {params.filter_dims}")
    if windows.c_in != params.c_in or (windows.h_f, windows.w_f, windows.stride) != (params.h_f, params.w_f,
                                                                                       params.stride):
        raise ShapeError("window tensor geometry does not match params")
    fd = f.data if f.device == windows.data.device else f.data.to(windows.data.device)
    out = torch.empty((windows.n, params.c_out, windows.h_out, windows.w_out), dtype=DTYPE,
                      device=windows.data.device)
    basic_windows_into(windows.data, fd, out, params)
    return Tensor4(out)


def conv_im2win_basic(inp, flt, params: ConvParams) -> Tensor4:
    """Window-order transform followed by one thread per output element (reference.py:222-225)."""
    i = inp if isinstance(inp, Tensor4) else Tensor4(inp)
    f = flt if isinstance(flt, Tensor4) else Tensor4(flt)
    check_conv_operands(i, f, params)
    return compute_from_windows_basic(im2win(i, params), f, params)


def cl_supported(c_in: int, variant: str) -> bool:
    """The channels-innermost TMA path needs c_in * element size to be a multiple of 16 bytes."""
    if variant == "tf32":
        return c_in % 4 == 0
    if variant == "bf16":
        return c_in % 8 == 0
    return False


def im2win_cl_shape(inp_dims: tuple[int, int, int, int], params: ConvParams) -> tuple[int, int, int, int]:
    """Shape of the channels-innermost window tensor: (N*Ho, w_eff, Hf, C)."""
    n_img, c_in, h_in, w_in = inp_dims
    h_out, w_out = output_dims(h_in, w_in, params)
    return (n_img * h_out, (w_out - 1) * params.stride + params.w_f, params.h_f, c_in)


def im2win_cl_into(src: torch.Tensor, dst: torch.Tensor, params: ConvParams) -> None:
    """Channels-innermost window transform (TC fast path); dst float32 or bfloat16."""
    n_img, c_in, h_in, w_in = (int(d) for d in src.shape)
    dtype = 1 if dst.dtype == torch.bfloat16 else 0
    with torch.cuda.device(src.device):
        rc = _lib.load().im2win_transform_cl(
            src.data_ptr(), dst.data_ptr(), n_img, c_in, h_in, w_in, params.h_f, params.w_f, params.stride, dtype,
            torch.cuda.current_stream(src.device).cuda_stream)
    _lib.check(rc)


def conv_cl_into(win_cl: torch.Tensor, flt: torch.Tensor, out: torch.Tensor, params: ConvParams,
                 variant: str) -> None:
    """tcgen05 convolution over the channels-innermost window tensor (TMA-fed)."""
    n_img, c_out, h_out, w_out = (int(d) for d in out.shape)
    code = _variant_code(variant)
    lib = _lib.load()
    nbytes = lib.im2win_conv_cl_workspace_bytes(params.c_in, params.c_out, params.h_f, params.w_f)
    stream = torch.cuda.current_stream(out.device).cuda_stream
    ws = _workspace(out.device, stream, nbytes)
    with torch.cuda.device(out.device):
        rc = lib.im2win_conv_cl(win_cl.data_ptr(), flt.data_ptr(), out.data_ptr(), n_img, params.c_in, c_out,
                                h_out, w_out, params.h_f, params.w_f, params.stride, code, ws.data_ptr(),
                                ws.numel(), stream)
    _lib.check(rc)


def nhwc_into(src: torch.Tensor, dst: torch.Tensor, pad: int = 0) -> None:
    """NCHW float32 -> channels-last copy (float32 or bfloat16) for the fused TC path.

    pad > 0: dst is (N, H + 2*pad, W + 2*pad, pitch) and its border pixels are zeroed.
    """
    n_img, c_in, h_in, w_in = (int(d) for d in src.shape)
    dtype = 1 if dst.dtype == torch.bfloat16 else 0
    with torch.cuda.device(src.device):
        rc = _lib.load().im2win_nchw_to_nhwc_padded(src.data_ptr(), dst.data_ptr(), n_img, c_in, h_in, w_in, dtype,
                                                    pad, torch.cuda.current_stream(src.device).cuda_stream)
    _lib.check(rc)


def nhwc_pitch(c_in: int, variant: str) -> int:
    """Channel pitch of the channels-last copy: the smallest 16-byte multiple >= c_in."""
    q = 8 if variant == "bf16" else 4
    return -(-c_in // q) * q


def conv_fused_into(x_nhwc: torch.Tensor, flt: torch.Tensor, out: torch.Tensor, params: ConvParams,
                    variant: str, ws: torch.Tensor | None = None) -> None:
    """tcgen05 convolution whose window tiles TMA builds from the channels-last input."""
    n_img, h_in, w_in, _pitch = (int(d) for d in x_nhwc.shape)
    c_in = params.c_in
    code = _variant_code(variant)
    lib = _lib.load()
    nbytes = lib.im2win_conv_fused_workspace_bytes(params.c_in, params.c_out, params.h_f, params.w_f)
    stream = torch.cuda.current_stream(out.device).cuda_stream
    ws = _workspace(out.device, stream, nbytes) if ws is None else _check_ws(ws, nbytes)
    with torch.cuda.device(out.device):
        rc = lib.im2win_conv_fused(x_nhwc.data_ptr(), flt.data_ptr(), out.data_ptr(), n_img, c_in, h_in, w_in,
                                   params.c_out, params.h_f, params.w_f, params.stride, code, ws.data_ptr(),
                                   ws.numel(), stream)
    _lib.check(rc)


def conv_fused_nchw_into(x: torch.Tensor, x_nhwc: torch.Tensor, flt: torch.Tensor, out: torch.Tensor,
                         params: ConvParams, variant: str, ws: torch.Tensor | None = None) -> None:
    """The fused tensor-core conv straight from the NCHW input: extra warps of the conv kernel
    write the channels-last scratch ``x_nhwc`` while the tensor cores consume it (no separate
    copy kernel).  Same bits as ``nhwc_into`` + ``conv_fused_into``."""
    n_img, c_in, h_in, w_in = (int(d) for d in x.shape)
    code = _variant_code(variant)
    lib = _lib.load()
    nbytes = lib.im2win_conv_fused_nchw_workspace_bytes(n_img, c_in, params.c_out, params.h_f, params.w_f)
    stream = torch.cuda.current_stream(out.device).cuda_stream
    ws = _workspace(out.device, stream, nbytes) if ws is None else _check_ws(ws, nbytes)
    with torch.cuda.device(out.device):
        rc = lib.im2win_conv_fused_nchw(x.data_ptr(), x_nhwc.data_ptr(), flt.data_ptr(), out.data_ptr(), n_img,
                                        c_in, h_in, w_in, params.c_out, params.h_f, params.w_f, params.stride, code,
                                        ws.data_ptr(), ws.numel(), stream)
    _lib.check(rc)


def feed_enabled(params: ConvParams) -> bool:
    """Whether the fused path goes through the one-call entry (im2win_conv_fused_nchw), where the
    library either produces the channels-last copy inside the conv kernel or runs its copy
    kernel first (rule and IM2WIN_FEED switch in conv_tc_fused.cu).  Zero padding keeps the
    two-call form, whose copy kernel writes the border."""
    return params.pad == 0


def direct_supported(inp_dims, params: ConvParams, variant: str) -> bool:
    """Whether the in-SM im2win tensor-core kernel (few-channel inputs) covers this shape."""
    if variant not in ("tf32", "bf16"):
        return False
    n_img, c_in, h_in, w_in = (int(d) for d in inp_dims)
    return bool(_lib.load().im2win_conv_direct_supported(n_img, c_in, h_in, w_in, params.c_out, params.h_f,
                                                         params.w_f, params.stride, params.pad,
                                                         _variant_code(variant)))


def direct_preferred(inp_dims, params: ConvParams, variant: str) -> bool:
    """The auto path's choice of the direct kernel (library rule im2win_conv_direct_preferred)."""
    if variant not in ("tf32", "bf16"):
        return False
    n_img, c_in, h_in, w_in = (int(d) for d in inp_dims)
    return bool(_lib.load().im2win_conv_direct_preferred(n_img, c_in, h_in, w_in, params.c_out, params.h_f,
                                                         params.w_f, params.stride, params.pad,
                                                         _variant_code(variant)))


def conv_direct_into(x: torch.Tensor, flt: torch.Tensor, out: torch.Tensor, params: ConvParams, variant: str,
                     ws: torch.Tensor | None = None) -> None:
    """tcgen05 convolution that builds the im2win windows in shared memory from the NCHW input."""
    n_img, c_in, h_in, w_in = (int(d) for d in x.shape)
    code = _variant_code(variant)
    lib = _lib.load()
    nbytes = lib.im2win_conv_direct_workspace(c_in, params.c_out, params.h_f, params.w_f, code)
    stream = torch.cuda.current_stream(out.device).cuda_stream
    ws = _workspace(out.device, stream, nbytes) if ws is None else _check_ws(ws, nbytes)
    with torch.cuda.device(out.device):
        rc = lib.im2win_conv_direct(x.data_ptr(), flt.data_ptr(), out.data_ptr(), n_img, c_in, h_in, w_in,
                                    params.c_out, params.h_f, params.w_f, params.stride, params.pad, code,
                                    ws.data_ptr(), ws.numel(), stream)
    _lib.check(rc)


TC_PATHS = ("auto", "direct", "fused", "cl", "gather")


def conv_im2win_opt(inp, flt, params: ConvParams, plan: TilePlan | None = None, *,
                    variant: str = "fp32-exact", tc_path: str = "auto") -> Tensor4:
    """Window-order transform followed by the tiled kernel (optimized.py:237-241).

    FP32 variants: the tiled kernel gathers every im2win window element straight from the
    NCHW input in the reference's k order (Ĩ[i,c,oh,(ow*s+fw)*Hf+fh] = X[i,c,oh*s+fh,ow*s+fw],
    layouts.py:73-83), so Ĩ is never written and the bits equal `im2win` followed by
    `compute_from_windows_opt`; with zero padding (or the micro_kernel=False ablation plan) the
    transform to Ĩ runs first, in image chunks above the window budget.  Tensor-core variants pick
    (tc_path="auto"): "direct" — for few-channel inputs (C <= 16) producer warps
    build each pixel's im2win window in shared memory from the NCHW input;
    "fused" — TMA builds window tiles from a channels-last copy
    of the input (no Ĩ); "cl" — materialised channels-innermost Ĩ streamed by TMA;
    "gather" — reference Ĩ gathered by producer warps.  The fused copy pads the
    channel pitch to a 16-byte multiple (zeros); "cl" needs c_in * element size
    to be a multiple of 16 bytes and otherwise falls back to gather.
    """
    if tc_path not in TC_PATHS:
        raise ValueError(f"tc_path must be one of {TC_PATHS}")
    i = inp if isinstance(inp, Tensor4) else Tensor4(inp)
    f = flt if isinstance(flt, Tensor4) else Tensor4(flt)
    h_out, w_out = check_conv_operands(i, f, params)
    ok = cl_supported(params.c_in, variant)
    use_direct = direct_supported(i.dims, params, variant) if tc_path == "direct" else (
        tc_path == "auto" and direct_preferred(i.dims, params, variant))
    if use_direct:
        out = torch.empty((i.dims[0], params.c_out, h_out, w_out), dtype=DTYPE, device=i.device)
        fd = f.data if f.device == i.device else f.data.to(i.device)
        conv_direct_into(i.data, fd, out, params, variant)
        return Tensor4(out)
    if tc_path == "direct":
        raise ValueError("tc_path='direct' does not cover this shape (needs C <= 16, Co <= 256)")
    if variant in ("tf32", "bf16") and tc_path in ("auto", "fused"):
        dt = torch.bfloat16 if variant == "bf16" else torch.float32
        n_img, c_in, h_in, w_in = i.dims
        pad = params.pad
        x_cl = torch.empty((n_img, h_in + 2 * pad, w_in + 2 * pad, nhwc_pitch(c_in, variant)), dtype=dt,
                           device=i.device)
        out = torch.empty((n_img, params.c_out, h_out, w_out), dtype=DTYPE, device=i.device)
        fd = f.data if f.device == i.device else f.data.to(i.device)
        if feed_enabled(params):
            conv_fused_nchw_into(i.data, x_cl, fd, out, params, variant)
        else:
            nhwc_into(i.data, x_cl, pad)
            conv_fused_into(x_cl, fd, out, params, variant)
        return Tensor4(out)
    if ok and tc_path == "cl" and params.pad:
        raise ValueError("tc_path='cl' has no zero padding; use 'fused' or 'gather'")
    if ok and tc_path == "cl":
        dt = torch.bfloat16 if variant == "bf16" else torch.float32
        win_cl = torch.empty(im2win_cl_shape(i.dims, params), dtype=dt, device=i.device)
        im2win_cl_into(i.data, win_cl, params)
        out = torch.empty((i.dims[0], params.c_out, h_out, w_out), dtype=DTYPE, device=i.device)
        fd = f.data if f.device == i.device else f.data.to(i.device)
        conv_cl_into(win_cl, fd, out, params, variant)
        return Tensor4(out)
    if variant in ("fp32-exact", "fp32-fma") and nchw_direct(params, plan):
        fd = f.data if f.device == i.device else f.data.to(i.device)
        out = torch.empty((i.dims[0], params.c_out, h_out, w_out), dtype=DTYPE, device=i.device)
        conv_nchw_into(i.data, fd, out, params, plan, variant)
        return Tensor4(out)
    return _fp32_chunked(i, f, params, plan, variant, h_out, w_out)


def nchw_direct(params: ConvParams, plan: TilePlan | None = None) -> bool:
    """Whether the FP32 conv_im2win_opt gathers its windows straight from the NCHW input
    (im2win_conv_nchw_f32, no Ĩ written; the default) rather than transforming to Ĩ first.
    Same bits either way.  Zero padding and the TilePlan(micro_kernel=False) ablation keep the
    Ĩ path; IM2WIN_FP32_PATH=windows forces it (A/B)."""
    if params.pad or (plan is not None and not plan.micro_kernel):
        return False
    return os.environ.get("IM2WIN_FP32_PATH", "nchw") != "windows"


def window_budget_bytes() -> int:
    """Largest im2win tensor conv_im2win_opt materialises at once (FP32 variants); larger
    batches are transformed and convolved in image chunks through one reused Ĩ buffer.
    IM2WIN_WINDOW_BUDGET (bytes; 0 = no limit), default 1 GiB."""
    return int(os.environ.get("IM2WIN_WINDOW_BUDGET", str(1 << 30)))


def _fp32_chunked(i: Tensor4, f: Tensor4, params: ConvParams, plan, variant: str, h_out: int,
                  w_out: int) -> Tensor4:
    """Transform + tiled conv; with Ĩ above the window budget, in image chunks.

    Images are independent (reference.py:78-90, the GEMM columns of different images never
    mix), so a chunk's transform + conv writes exactly the output rows the full-batch call
    would, with the same bits.  Peak extra memory: one chunk's Ĩ instead of the batch's
    (conv4 at N=128: 1.0 GB instead of 5.6 GB).  A chunk is at least 8 images so the conv
    grid still fills the GPU.
    """
    from .layouts import effective_width, im2win_into

    n_img = i.dims[0]
    w_eff = effective_width(w_out, params.w_f, params.stride)
    per_img = params.c_in * h_out * params.h_f * w_eff * 4
    budget = window_budget_bytes()
    if budget <= 0 or per_img * n_img <= budget:
        return compute_from_windows_opt(im2win(i, params), f, params, plan, variant=variant)
    chunk = max(8, budget // per_img)
    fd = f.data if f.device == i.device else f.data.to(i.device)
    out = torch.empty((n_img, params.c_out, h_out, w_out), dtype=DTYPE, device=i.device)
    win = torch.empty((min(chunk, n_img), params.c_in, h_out, params.h_f * w_eff), dtype=DTYPE, device=i.device)
    for lo in range(0, n_img, chunk):
        hi = min(n_img, lo + chunk)
        wv = win[: hi - lo]
        im2win_into(i.data[lo:hi], wv, params)
        conv_windows_into(wv, fd, out[lo:hi], params, w_eff, plan, variant)
    return Tensor4(out)


def _host_f32(x, ndim: int) -> torch.Tensor:
    """A host operand as a contiguous float32 CPU tensor (no copy when it already is one)."""
    if isinstance(x, Tensor4):
        raise ShapeError("conv_im2win_opt_host takes host operands; use conv_im2win_opt for device tensors")
    if hasattr(x, "data") and isinstance(getattr(x, "data"), np.ndarray):
        x = x.data  # a reference winconv.Tensor4 (or look-alike)
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    if not isinstance(x, torch.Tensor):
        raise ShapeError(f"unsupported operand type {type(x).__name__}")
    if x.is_cuda:
        raise ShapeError("conv_im2win_opt_host takes host operands; use conv_im2win_opt for device tensors")
    if x.dim() != ndim:
        raise ShapeError(f"expected a {ndim}-D array, got {x.dim()}-D")
    if min(x.shape) < 1:
        raise ShapeError(f"all extents must be positive, got {tuple(x.shape)}")
    return x.to(DTYPE).contiguous()


class HostConv:
    """A submitted host-buffer convolution (conv_im2win_opt_host(..., wait=False)).

    Holds the operands and the device workspace until `wait()` returns; `out`
    is valid after that.  Dropping an unfinished handle waits for it.
    """

    def __init__(self, out, ticket, keep):
        self.out = out
        self._ticket = ticket
        self._keep = keep

    def wait(self) -> torch.Tensor:
        if self._keep is not None:
            rc = _lib.load().im2win_conv_host_wait(self._ticket)
            self._keep = None
            _lib.check(rc)
        return self.out

    def __del__(self):
        if getattr(self, "_keep", None) is not None:
            _lib.load().im2win_conv_host_wait(self._ticket)


class _MultiHostConv:
    """Handles of one host convolution split across several GPUs (batch slices)."""

    def __init__(self, out, parts):
        self.out = out
        self._parts = parts

    def wait(self) -> torch.Tensor:
        for h in self._parts:
            h.wait()
        self._parts = []
        return self.out


def conv_im2win_opt_host(inp, flt, params: ConvParams, plan: TilePlan | None = None, *,
                         variant: str = "fp32-exact", out: torch.Tensor | None = None, chunk_images: int = 0,
                         device=None, devices=None, wait: bool = True):
    """`conv_im2win_opt` for host operands, as the reference is called (optimized.py:237-241).

    Host input and filter in, host output back (a CPU float32 tensor; pass a
    page-locked `out` to reuse it).  The library cuts the batch into chunks and
    overlaps upload, transform + conv, and download on three streams
    (csrc/pipeline.cu); results are bit-identical to the device path.  Page-locked
    operands let the copies overlap; pageable ones work but serialise.
    With wait=False the call returns a `HostConv` at once; consecutive
    submissions overlap each other (uploads of one with downloads of the last).
    `devices` (a list of CUDA devices) splits the batch into contiguous slices, one
    per device, each streamed over its own PCIe link from one process (images are
    independent, reference.py:78-90, so the result is bit-identical to one device).
    """
    if devices is not None and len(devices) > 1:
        from .sharding import shard_bounds

        x = _host_f32(inp, 4)
        f = _host_f32(flt, 4)
        n_img = int(x.shape[0])
        if out is None:
            h_out, w_out = output_dims(int(x.shape[2]), int(x.shape[3]), params)
            out = torch.empty((n_img, params.c_out, h_out, w_out), dtype=DTYPE, pin_memory=True)
        parts = []
        for r, d in enumerate(devices):
            lo, hi = shard_bounds(n_img, len(devices), r)
            if hi > lo:
                parts.append(conv_im2win_opt_host(x[lo:hi], f, params, plan, variant=variant, out=out[lo:hi],
                                                  chunk_images=chunk_images, device=d, wait=False))
        handle = _MultiHostConv(out, parts)
        return handle.wait() if wait else handle
    x = _host_f32(inp, 4)
    f = _host_f32(flt, 4)
    n_img, c_in, h_in, w_in = (int(d) for d in x.shape)
    if tuple(f.shape) != params.filter_dims:
        raise ShapeError(f"filter dims {tuple(f.shape)} do not match params {params.filter_dims}")
    if c_in != params.c_in:
        raise ShapeError(f"input has {c_in} channels, params expect {params.c_in}")
    h_out, w_out = output_dims(h_in, w_in, params)
    shape = (n_img, params.c_out, h_out, w_out)
    if out is None:
        out = torch.empty(shape, dtype=DTYPE, pin_memory=True)
    elif tuple(out.shape) != shape or out.dtype != DTYPE or out.is_cuda or not out.is_contiguous():
        raise ShapeError(f"out must be a contiguous float32 host tensor of shape {shape}")
    if not torch.cuda.is_available():
        raise ShapeError("a CUDA device is required (this package has no CPU path)")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    code = _variant_code(variant)
    lib = _lib.load()
    nbytes = lib.im2win_conv_host_workspace_bytes(n_img, c_in, h_in, w_in, params.c_out, params.h_f, params.w_f,
                                                  params.stride, params.pad, code, chunk_images)
    stream = torch.cuda.current_stream(dev).cuda_stream
    cplan = to_c_plan(plan)
    cp = None if cplan is None else _byref(cplan)
    args = (x.data_ptr(), f.data_ptr(), out.data_ptr(), n_img, c_in, h_in, w_in, params.c_out, params.h_f,
            params.w_f, params.stride, params.pad, cp, code, chunk_images)
    if wait:
        # per call (torch's caching allocator recycles it): the chunk buffers can be GBs at large N,
        # so they are not pinned in the module-level workspace cache the device entry points share
        ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
        _lib.check(lib.im2win_conv_host_f32(*args, ws.data_ptr(), ws.numel(), stream))
        return out
    import ctypes

    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)  # owned by the handle until wait()
    ticket = ctypes.c_int64(-1)
    _lib.check(lib.im2win_conv_host_submit(*args, ws.data_ptr(), ws.numel(), stream, ctypes.byref(ticket)))
    return HostConv(out, ticket.value, (x, f, ws, cplan))


def conv_im2win_opt_host_batch(jobs, *, variant: str = "fp32-exact", outs=None, chunk_images: int = 0,
                               device=None, devices=None) -> list:
    """Several independent host-operand convolutions (e.g. the layers of a benchmark step).

    `jobs` is a list of (inp, flt, params); `outs` optional page-locked outputs in the same
    order.  All jobs are submitted non-blocking to the streamed host pipeline, ordered so
    the PCIe download engine starts early: jobs that download more than they upload go
    first, upload-heavy jobs last (uploads of one job overlap downloads of the ones before
    it).  Returns the host outputs in the order of `jobs`.
    """
    def elems(x):
        return int(np.prod(x.shape)) if hasattr(x, "shape") else int(np.prod(x.data.shape))

    balance = []
    for inp, flt, params in jobs:
        shape = inp.shape if hasattr(inp, "shape") else inp.data.shape
        h_out, w_out = output_dims(int(shape[2]), int(shape[3]), params)
        d2h = int(shape[0]) * params.c_out * h_out * w_out
        balance.append(d2h - elems(inp))
    order = sorted(range(len(jobs)), key=lambda i: -balance[i])
    handles = [None] * len(jobs)
    for i in order:
        inp, flt, params = jobs[i]
        handles[i] = conv_im2win_opt_host(inp, flt, params, variant=variant, chunk_images=chunk_images,
                                          out=None if outs is None else outs[i], device=device, devices=devices,
                                          wait=False)
    return [h.wait() for h in handles]


class CapturedConv:
    """A fixed-shape im2win convolution captured once in a CUDA graph and replayed.

    For serving loops that call the same layer repeatedly: the transform (or the
    channels-last copy) and the convolution are recorded with their buffers,
    workspace and tensor maps, so each call is one graph launch instead of several
    Python -> C ABI -> kernel launches.  Call with a new input (and optionally a new
    filter) of the captured shapes; the result is written into `self.out` (a device
    tensor reused across calls; clone it to keep it).  Bit-identical to
    `conv_im2win_opt` with the same arguments.
    """

    def __init__(self, input_shape, params: ConvParams, flt=None, plan: TilePlan | None = None, *,
                 variant: str = "fp32-exact", device=None):
        n_img, c_in, h_in, w_in = (int(d) for d in input_shape)
        if c_in != params.c_in:
            raise ShapeError(f"input has {c_in} channels, params expect {params.c_in}")
        _variant_code(variant)
        if not torch.cuda.is_available():
            raise ShapeError("a CUDA device is required (this package has no CPU path)")
        self.device = torch.device(device) if device is not None else torch.device("cuda",
                                                                                    torch.cuda.current_device())
        self.params, self.variant = params, variant
        h_out, w_out = output_dims(h_in, w_in, params)
        dev = self.device
        self.input = torch.zeros((n_img, c_in, h_in, w_in), dtype=DTYPE, device=dev)
        self.filter = torch.zeros(params.filter_dims, dtype=DTYPE, device=dev)
        if flt is not None:
            self.filter.copy_(Tensor4(flt).data)
        self.out = torch.empty((n_img, params.c_out, h_out, w_out), dtype=DTYPE, device=dev)
        # the graph keeps pointing at its workspace: it is owned here, not taken from the shared cache
        lib = _lib.load()
        code = _variant_code(variant)
        ws_bytes = max(lib.im2win_conv_workspace_bytes(c_in, params.c_out, params.h_f, params.w_f, code),
                       lib.im2win_conv_fused_nchw_workspace_bytes(n_img, c_in, params.c_out, params.h_f, params.w_f),
                       lib.im2win_conv_direct_workspace(c_in, params.c_out, params.h_f, params.w_f, code))
        self._ws = torch.empty(max(ws_bytes, 1 << 16), dtype=torch.uint8, device=dev)
        if variant in ("tf32", "bf16") and direct_preferred(self.input.shape, params, variant):
            def body():
                conv_direct_into(self.input, self.filter, self.out, params, variant, self._ws)
        elif variant in ("tf32", "bf16"):
            dt = torch.bfloat16 if variant == "bf16" else torch.float32
            pad = params.pad
            self._mid = torch.empty((n_img, h_in + 2 * pad, w_in + 2 * pad, nhwc_pitch(c_in, variant)), dtype=dt,
                                    device=dev)

            if feed_enabled(params):
                def body():
                    conv_fused_nchw_into(self.input, self._mid, self.filter, self.out, params, variant, self._ws)
            else:
                def body():
                    nhwc_into(self.input, self._mid, pad)
                    conv_fused_into(self._mid, self.filter, self.out, params, variant, self._ws)
        elif nchw_direct(params, plan):
            def body():
                conv_nchw_into(self.input, self.filter, self.out, params, plan, variant, self._ws)
        else:
            from .layouts import effective_width, im2win_into

            w_eff = effective_width(w_out, params.w_f, params.stride)
            self._mid = torch.empty((n_img, c_in, h_out, params.h_f * w_eff), dtype=DTYPE, device=dev)

            def body():
                im2win_into(self.input, self._mid, params)
                conv_windows_into(self._mid, self.filter, self.out, params, w_eff, plan, variant, self._ws)

        # warm up on a side stream (allocates the workspace, sets kernel attributes), then capture
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.device(dev), torch.cuda.stream(side):
            body()
            self.kernel = _lib.last_kernel()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=side, capture_error_mode="relaxed"):
                body()
        torch.cuda.current_stream(dev).wait_stream(side)

    def __call__(self, inp, flt=None) -> Tensor4:
        """Copy the operands into the captured buffers and replay (on the current stream)."""
        x = inp.data if isinstance(inp, Tensor4) else inp
        if not isinstance(x, torch.Tensor):
            x = Tensor4(x).data
        if tuple(x.shape) != tuple(self.input.shape):
            raise ShapeError(f"input shape {tuple(x.shape)} differs from the captured {tuple(self.input.shape)}")
        self.input.copy_(x, non_blocking=True)
        if flt is not None:
            fd = flt.data if isinstance(flt, Tensor4) else flt
            if not isinstance(fd, torch.Tensor):
                fd = Tensor4(fd).data
            if tuple(fd.shape) != tuple(self.filter.shape):
                raise ShapeError(f"filter dims {tuple(fd.shape)} do not match params {self.params.filter_dims}")
            self.filter.copy_(fd, non_blocking=True)
        self.graph.replay()
        return Tensor4(self.out)
