"""Operand carrier, convolution geometry and parity metrics (device side).

Mirrors winconv `tensors.py` (/root/reference/pkg/src/winconv/tensors.py):
`ConvParams` (:94-112), `output_dims` (:115-123), `check_conv_operands`
(:126-132), `Tensor4` (:28-50) and `max_rel_diff` (:135-150).  The difference
is where the data lives: a `Tensor4` here wraps a float32, C-contiguous, 4-D
**CUDA** `torch.Tensor`.  Host data (numpy arrays, reference `Tensor4`s, CPU
tensors) is accepted at the boundary and uploaded once; nothing computes on
the CPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import GeometryError, ShapeError

DTYPE = torch.float32


def _to_device_f32(data, ndim: int, device=None) -> torch.Tensor:
    """Coerce an operand into a contiguous float32 CUDA tensor (tensors.py:19-25)."""
    if isinstance(data, Tensor4):
        data = data.data
    elif hasattr(data, "data") and isinstance(getattr(data, "data"), np.ndarray):
        data = data.data  # a reference winconv.Tensor4 (or look-alike)
    if isinstance(data, np.ndarray):
        data = torch.from_numpy(np.ascontiguousarray(data, dtype=np.float32))
    if not isinstance(data, torch.Tensor):
        raise ShapeError(f"unsupported operand type {type(data).__name__}")
    if data.dim() != ndim:
        raise ShapeError(f"expected a {ndim}-D array, got {data.dim()}-D")
    if min(data.shape) < 1:
        raise ShapeError(f"all extents must be positive, got {tuple(data.shape)}")
    if data.dtype != DTYPE:
        data = data.to(DTYPE)
    if not data.is_cuda:
        if not torch.cuda.is_available():
            raise ShapeError("a CUDA device is required (this package has no CPU path)")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        data = data.to(dev)
    return data.contiguous()


@dataclass(frozen=True, eq=False)
class Tensor4:
    """Contiguous 4-D float32 CUDA tensor; carrier for inputs, filters, outputs."""

    data: torch.Tensor

    def __post_init__(self):
        object.__setattr__(self, "data", _to_device_f32(self.data, 4))

    @property
    def dims(self) -> tuple[int, int, int, int]:
        return tuple(int(d) for d in self.data.shape)

    @property
    def device(self) -> torch.device:
        return self.data.device

    @classmethod
    def zeros(cls, d0: int, d1: int, d2: int, d3: int, device=None) -> "Tensor4":
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        return cls(torch.zeros((d0, d1, d2, d3), dtype=DTYPE, device=dev))

    def numpy(self) -> np.ndarray:
        """Host copy (synchronous device->host read)."""
        return self.data.detach().cpu().numpy()

    def __eq__(self, other) -> bool:
        """Bitwise equality, like the reference (tensors.py:45-50): +0 != -0, equal NaN bits match."""
        if not isinstance(other, Tensor4):
            return NotImplemented
        if self.dims != other.dims:
            return False
        b = other.data.to(self.data.device)
        return bool(torch.equal(self.data.view(torch.int32), b.view(torch.int32)))

    __hash__ = None


@dataclass(frozen=True)
class ConvParams:
    """Filter geometry plus a single stride applied to both spatial axes (tensors.py:94-112).

    `pad` (extension, default 0 = the reference's unpadded convolution) zero-pads the
    input by `pad` on every side inside the transform; the padded input is never
    materialised and the result is bit-identical to convolving an explicitly padded input.
    """

    c_in: int
    c_out: int
    h_f: int
    w_f: int
    stride: int = 1
    pad: int = 0

    def __post_init__(self):
        for name in ("c_in", "c_out", "h_f", "w_f", "stride"):
            value = getattr(self, name)
            if int(value) != value or value < 1:
                raise GeometryError(f"{name} must be a positive integer, got {value}")
        if int(self.pad) != self.pad or self.pad < 0:
            raise GeometryError(f"pad must be a non-negative integer, got {self.pad}")

    @property
    def filter_dims(self) -> tuple[int, int, int, int]:
        return (self.c_out, self.c_in, self.h_f, self.w_f)


def output_dims(h_in: int, w_in: int, params: ConvParams) -> tuple[int, int]:
    """Output extents: floor((in + 2*pad - filter) / stride) + 1 per axis (tensors.py:115-123, pad = 0)."""
    h_in, w_in = h_in + 2 * params.pad, w_in + 2 * params.pad
    if params.h_f > h_in or params.w_f > w_in:
        raise GeometryError(
            f"filter {params.h_f}x{params.w_f} larger than input {h_in}x{w_in}"
        )
    h_out = (h_in - params.h_f) // params.stride + 1
    w_out = (w_in - params.w_f) // params.stride + 1
    return h_out, w_out


def check_conv_operands(inp: Tensor4, flt: Tensor4, params: ConvParams) -> tuple[int, int]:
    """Validate input/filter/params consistency; returns the output extents (tensors.py:126-132)."""
    if flt.dims != params.filter_dims:
        raise ShapeError(f"filter dims {flt.dims} do not match params {params.filter_dims}")
    if inp.dims[1] != params.c_in:
        raise ShapeError(f"input has {inp.dims[1]} channels, params expect {params.c_in}")
    return output_dims(inp.dims[2], inp.dims[3], params)


def _as_host_f32(t) -> np.ndarray:
    if isinstance(t, Tensor4):
        return t.numpy()
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy().astype(np.float32, copy=False)
    if hasattr(t, "data") and isinstance(t.data, np.ndarray):
        return t.data
    return np.asarray(t, dtype=np.float32)


def max_rel_diff(a, b) -> float:
    """max over elements of |a-b| / max(|a|, |b|, 1), identical bits -> 0 (tensors.py:135-150).

    Host-side parity metric; accepts device Tensor4s, torch tensors or numpy arrays.
    """
    x32 = np.ascontiguousarray(_as_host_f32(a), dtype=np.float32)
    y32 = np.ascontiguousarray(_as_host_f32(b), dtype=np.float32)
    if x32.shape != y32.shape:
        raise ShapeError(f"dims differ: {x32.shape} vs {y32.shape}")
    x = x32.astype(np.float64)
    y = y32.astype(np.float64)
    denom = np.maximum(np.maximum(np.abs(x), np.abs(y)), 1.0)
    with np.errstate(invalid="ignore"):
        diff = np.abs(x - y) / denom
    diff[x32.view(np.uint32) == y32.view(np.uint32)] = 0.0
    return float(np.max(diff)) if diff.size else 0.0


def normalized_max_diff(a, b) -> float:
    """max|a-b| / rms(b): the tolerance metric for the TF32/BF16 tensor-core variants.

    The reference's floor-1 metric is dominated by element magnitude for
    reduced-precision operands; normalizing by the RMS of the
    reference output makes the bound independent of K.
    """
    x = _as_host_f32(a).astype(np.float64)
    y = _as_host_f32(b).astype(np.float64)
    if x.shape != y.shape:
        raise ShapeError(f"dims differ: {x.shape} vs {y.shape}")
    rms = float(np.sqrt(np.mean(y * y))) if y.size else 0.0
    return float(np.max(np.abs(x - y))) / max(rms, 1e-30)
