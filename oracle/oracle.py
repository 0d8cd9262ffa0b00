"""CPU oracle for the im2win path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` arm may import this module; the product package never
does.  It wraps the plain-C restatement in im2win_oracle.c:

  im2win_fill          <- winconv layouts.py:73-83 (_im2win_fill)
  conv_direct          <- winconv kernels/reference.py:70-90 (_direct_kernel),
                          float32 unfused multiply-add, ascending k
  conv_from_windows    <- winconv kernels/reference.py:180-206 (_basic_window_kernel)

Parity is pinned: tests/test_oracle.py checks these functions against the
golden vectors in tests/golden/ that tests/golden/make_golden.py produced by
running the reference package itself.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> Path:
    src = HERE / "im2win_oracle.c"
    if force or not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE), "-B", "liboracle.so"], check=True)
    return LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(str(LIB))
            i64, i32, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
            lib.oracle_im2win_fill.argtypes = [vp, vp, i64, i64, i64, i64, i32, i32, i32, i32]
            lib.oracle_conv_direct.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i32, i32, i32, i32]
            lib.oracle_conv_from_windows.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i64, i32, i32,
                                                     i32, i32]
            lib.oracle_max_threads.restype = i32
            _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def _threads(threads: int | None) -> int:
    if threads is None:
        return int(os.environ.get("ORACLE_THREADS", max_threads()))
    return threads


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def out_dims(h: int, w: int, hf: int, wf: int, s: int) -> tuple[int, int]:
    return (h - hf) // s + 1, (w - wf) // s + 1


def im2win_fill(inp: np.ndarray, hf: int, wf: int, s: int, threads: int | None = None) -> np.ndarray:
    x = _f32(inp)
    n, c, h, w = x.shape
    ho, wo = out_dims(h, w, hf, wf, s)
    w_eff = (wo - 1) * s + wf
    dst = np.empty((n, c, ho, hf * w_eff), dtype=np.float32)
    _load().oracle_im2win_fill(x.ctypes.data, dst.ctypes.data, n, c, h, w, hf, wf, s, _threads(threads))
    return dst


def conv_direct(inp: np.ndarray, flt: np.ndarray, s: int, threads: int | None = None) -> np.ndarray:
    x = _f32(inp)
    f = _f32(flt)
    n, c, h, w = x.shape
    co, ci, hf, wf = f.shape
    assert ci == c
    ho, wo = out_dims(h, w, hf, wf, s)
    out = np.empty((n, co, ho, wo), dtype=np.float32)
    _load().oracle_conv_direct(x.ctypes.data, f.ctypes.data, out.ctypes.data, n, c, h, w, co, hf, wf, s,
                               _threads(threads))
    return out


def conv_from_windows(win: np.ndarray, flt: np.ndarray, s: int, w_out: int,
                      threads: int | None = None) -> np.ndarray:
    wnd = _f32(win)
    f = _f32(flt)
    n, c, ho, row_len = wnd.shape
    co, ci, hf, wf = f.shape
    assert ci == c
    out = np.empty((n, co, ho, w_out), dtype=np.float32)
    _load().oracle_conv_from_windows(wnd.ctypes.data, f.ctypes.data, out.ctypes.data, n, c, ho, w_out,
                                     row_len, co, hf, wf, s, _threads(threads))
    return out


def checksum(a: np.ndarray) -> str:
    """sha256[:16] of the raw float32 bytes (winconv bench.py:148-149)."""
    import hashlib

    return hashlib.sha256(_f32(a).tobytes()).hexdigest()[:16]
