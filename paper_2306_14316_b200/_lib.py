"""ctypes binding of libim2win_sm100.so (the C ABI in include/im2win_sm100.h).

There is no fallback: if the shared library is missing or cannot be loaded,
every entry point raises.  Only plain pointers, integers and a stream handle
cross the boundary.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import KernelError

LIB_PATH = Path(__file__).resolve().parent / "libim2win_sm100.so"

# enum im2win_variant
FP32_EXACT = 0
FP32_FMA = 1
TF32 = 2
BF16 = 3
VARIANTS = {"fp32-exact": FP32_EXACT, "fp32-fma": FP32_FMA, "tf32": TF32, "bf16": BF16}

# every symbol include/im2win_sm100.h declares
EXPORTED_SYMBOLS = (
    "im2win_transform_f32",
    "im2win_transform_f32_padded",
    "im2win_conv_workspace_bytes",
    "im2win_conv_f32",
    "im2win_conv_nchw_f32",
    "im2win_last_error",
    "im2win_last_kernel",
    "im2win_conv_launch_count",
    "im2win_abi_version",
    "im2win_bench_fp32_peak",
    "im2win_transform_cl",
    "im2win_conv_cl_workspace_bytes",
    "im2win_conv_cl",
    "im2win_nchw_to_nhwc",
    "im2win_nchw_to_nhwc_padded",
    "im2win_conv_fused_workspace_bytes",
    "im2win_conv_fused",
    "im2win_conv_fused_nchw_workspace_bytes",
    "im2win_conv_fused_nchw",
    "im2win_conv_basic_f32",
    "im2win_conv_direct_supported",
    "im2win_conv_direct_preferred",
    "im2win_conv_direct_workspace",
    "im2win_conv_direct",
    "im2win_conv_host_workspace_bytes",
    "im2win_conv_host_f32",
    "im2win_conv_host_submit",
    "im2win_conv_host_wait",
)


class TilePlanC(ctypes.Structure):
    _fields_ = [
        ("block_cfg", ctypes.c_int32),
        ("micro_kernel", ctypes.c_int32),
        ("vectorized_load", ctypes.c_int32),
        ("prefetch_double_buffer", ctypes.c_int32),
    ]


_lock = threading.Lock()
_lib = None


def load(path: Path | str | None = None) -> ctypes.CDLL:
    """Load (once) and type the library; raises if it is absent."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        # IM2WIN_LIB: an alternate build of the same library (exploration builds, tools/build_variant.sh)
        p = Path(path) if path is not None else Path(os.environ.get("IM2WIN_LIB", LIB_PATH))
        if not p.exists():
            raise ImportError(
                f"{p} is missing: build it with `python -m paper_2306_14316_b200.build` "
                "(this package has no CPU fallback)"
            )
        lib = ctypes.CDLL(str(p))
        i64, i32, vp, sz = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t
        lib.im2win_transform_f32.argtypes = [vp, vp, i64, i64, i64, i64, i32, i32, i32, vp]
        lib.im2win_transform_f32.restype = ctypes.c_int
        lib.im2win_transform_f32_padded.argtypes = [vp, vp, i64, i64, i64, i64, i32, i32, i32, i32, vp]
        lib.im2win_transform_f32_padded.restype = ctypes.c_int
        lib.im2win_conv_workspace_bytes.argtypes = [i64, i64, i32, i32, i32]
        lib.im2win_conv_workspace_bytes.restype = sz
        lib.im2win_conv_f32.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i64, i32, i32, i32,
                                        ctypes.POINTER(TilePlanC), i32, vp, sz, vp]
        lib.im2win_conv_f32.restype = ctypes.c_int
        lib.im2win_conv_nchw_f32.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i32, i32, i32,
                                             ctypes.POINTER(TilePlanC), i32, vp, sz, vp]
        lib.im2win_conv_nchw_f32.restype = ctypes.c_int
        lib.im2win_last_error.argtypes = []
        lib.im2win_last_error.restype = ctypes.c_char_p
        lib.im2win_last_kernel.argtypes = []
        lib.im2win_last_kernel.restype = ctypes.c_char_p
        lib.im2win_conv_launch_count.argtypes = []
        lib.im2win_conv_launch_count.restype = ctypes.c_int64
        lib.im2win_abi_version.argtypes = []
        lib.im2win_abi_version.restype = ctypes.c_int32
        lib.im2win_bench_fp32_peak.argtypes = [vp, i32, i32, i32, vp]
        lib.im2win_bench_fp32_peak.restype = ctypes.c_int
        lib.im2win_transform_cl.argtypes = [vp, vp, i64, i64, i64, i64, i32, i32, i32, i32, vp]
        lib.im2win_transform_cl.restype = ctypes.c_int
        lib.im2win_conv_cl_workspace_bytes.argtypes = [i64, i64, i32, i32]
        lib.im2win_conv_cl_workspace_bytes.restype = sz
        lib.im2win_conv_cl.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i32, i32, i32, i32, vp, sz, vp]
        lib.im2win_conv_cl.restype = ctypes.c_int
        lib.im2win_nchw_to_nhwc.argtypes = [vp, vp, i64, i64, i64, i64, i32, vp]
        lib.im2win_nchw_to_nhwc.restype = ctypes.c_int
        lib.im2win_nchw_to_nhwc_padded.argtypes = [vp, vp, i64, i64, i64, i64, i32, i32, vp]
        lib.im2win_nchw_to_nhwc_padded.restype = ctypes.c_int
        lib.im2win_conv_fused_workspace_bytes.argtypes = [i64, i64, i32, i32]
        lib.im2win_conv_fused_workspace_bytes.restype = sz
        lib.im2win_conv_fused.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i32, i32, i32, i32, vp, sz, vp]
        lib.im2win_conv_fused.restype = ctypes.c_int
        lib.im2win_conv_fused_nchw_workspace_bytes.argtypes = [i64, i64, i64, i32, i32]
        lib.im2win_conv_fused_nchw_workspace_bytes.restype = sz
        lib.im2win_conv_fused_nchw.argtypes = [vp, vp, vp, vp, i64, i64, i64, i64, i64, i32, i32, i32, i32, vp, sz,
                                               vp]
        lib.im2win_conv_fused_nchw.restype = ctypes.c_int
        lib.im2win_conv_basic_f32.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i64, i32, i32, i32, vp]
        lib.im2win_conv_basic_f32.restype = ctypes.c_int
        lib.im2win_conv_direct_supported.argtypes = [i64, i64, i64, i64, i64, i32, i32, i32, i32, i32]
        lib.im2win_conv_direct_supported.restype = ctypes.c_int32
        lib.im2win_conv_direct_preferred.argtypes = [i64, i64, i64, i64, i64, i32, i32, i32, i32, i32]
        lib.im2win_conv_direct_preferred.restype = ctypes.c_int32
        lib.im2win_conv_direct_workspace.argtypes = [i64, i64, i32, i32, i32]
        lib.im2win_conv_direct_workspace.restype = sz
        lib.im2win_conv_direct.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i32, i32, i32, i32, i32, vp, sz, vp]
        lib.im2win_conv_direct.restype = ctypes.c_int
        lib.im2win_conv_host_workspace_bytes.argtypes = [i64, i64, i64, i64, i64, i32, i32, i32, i32, i32, i64]
        lib.im2win_conv_host_workspace_bytes.restype = sz
        lib.im2win_conv_host_f32.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i32, i32, i32, i32,
                                             ctypes.POINTER(TilePlanC), i32, i64, vp, sz, vp]
        lib.im2win_conv_host_f32.restype = ctypes.c_int
        lib.im2win_conv_host_submit.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i32, i32, i32, i32,
                                                ctypes.POINTER(TilePlanC), i32, i64, vp, sz, vp,
                                                ctypes.POINTER(ctypes.c_int64)]
        lib.im2win_conv_host_submit.restype = ctypes.c_int
        lib.im2win_conv_host_wait.argtypes = [i64]
        lib.im2win_conv_host_wait.restype = ctypes.c_int
        if path is None:
            _lib = lib
        return lib


def last_kernel() -> str:
    """Which kernel variant the last conv call on this thread launched (library-reported)."""
    return load().im2win_last_kernel().decode()


def check(rc: int) -> None:
    if rc != 0:
        msg = load().im2win_last_error().decode(errors="replace")
        raise KernelError(f"CUDA library error {rc}: {msg}")
