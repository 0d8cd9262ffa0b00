"""GEMM index space and tile plans.

`GemmDims` + `decompose_n/compose_n/decompose_k/compose_k` mirror
/root/reference/pkg/src/winconv/kernels/reference.py:30-67; `TilePlan` and
`default_plan` mirror kernels/plan.py:11-72 with the same validation
(PlanError) and the same toggle semantics.

On the GPU a plan selects among tile shapes compiled into
libim2win_sm100.so: the three toggles are honoured exactly
(micro_kernel=False -> one output per thread, vectorized_load=False ->
scalar shared-memory fragment loads, prefetch_double_buffer=False -> a
single-stage staging buffer); the block extents (m_b, n_b) select a compiled
CTA tile when they name one, otherwise the library's shape-based choice is
used.  Every plan yields bitwise-identical results (ascending-k float32
accumulation per element is plan independent, plan.py / optimized.py:11-16).
"""

from __future__ import annotations

from dataclasses import dataclass, replace

from .errors import PlanError, ShapeError
from .tensors import ConvParams, output_dims


@dataclass(frozen=True)
class GemmDims:
    """The M/N/K iteration space shared by the GEMM-shaped kernels (reference.py:30-46)."""

    m: int  # output channels
    n: int  # batch * output rows * output cols
    k: int  # input channels * filter rows * filter cols

    @classmethod
    def from_conv(cls, inp_dims: tuple[int, int, int, int], params: ConvParams) -> "GemmDims":
        if inp_dims[1] != params.c_in:
            raise ShapeError(f"input has {inp_dims[1]} channels, params expect {params.c_in}")
        h_out, w_out = output_dims(inp_dims[2], inp_dims[3], params)
        return cls(params.c_out, inp_dims[0] * h_out * w_out, params.c_in * params.h_f * params.w_f)


def decompose_n(n: int, h_out: int, w_out: int) -> tuple[int, int, int]:
    hw = h_out * w_out
    return n // hw, (n % hw) // w_out, (n % hw) % w_out


def compose_n(i_n: int, o_h: int, o_w: int, h_out: int, w_out: int) -> int:
    return (i_n * h_out + o_h) * w_out + o_w


def decompose_k(k: int, h_f: int, w_f: int) -> tuple[int, int, int]:
    fhw = h_f * w_f
    k_res = k % fhw
    return k // fhw, k_res // w_f, k_res % w_f


def compose_k(i_c: int, f_h: int, f_w: int, h_f: int, w_f: int) -> int:
    return (i_c * h_f + f_h) * w_f + f_w


@dataclass(frozen=True)
class TilePlan:
    """Block extents (m_b, n_b, k_b), per-thread micro-tile (m_t, n_t), three toggles (plan.py:11-48)."""

    m_b: int
    n_b: int
    k_b: int
    m_t: int
    n_t: int
    micro_kernel: bool = True
    vectorized_load: bool = True
    prefetch_double_buffer: bool = True

    def __post_init__(self):
        if not self.micro_kernel:
            object.__setattr__(self, "m_t", 1)
            object.__setattr__(self, "n_t", 1)
        for name in ("m_b", "n_b", "k_b", "m_t", "n_t"):
            value = getattr(self, name)
            if int(value) != value or value < 1:
                raise PlanError(f"{name} must be a positive integer, got {value}")
        if self.m_b % self.m_t:
            raise PlanError(f"m_t={self.m_t} does not divide m_b={self.m_b}")
        if self.n_b % self.n_t:
            raise PlanError(f"n_t={self.n_t} does not divide n_b={self.n_b}")

    @property
    def workers_per_block(self) -> int:
        return (self.m_b // self.m_t) * (self.n_b // self.n_t)

    def with_toggles(self, **kwargs) -> "TilePlan":
        return replace(self, **kwargs)


def _round_up(value: int, multiple: int) -> int:
    return ((value + multiple - 1) // multiple) * multiple


def default_plan(dims: GemmDims) -> TilePlan:
    """The reference's CPU blocking heuristic (plan.py:55-72), kept for API parity."""
    if min(dims.m, dims.n, dims.k) < 1:
        raise PlanError(f"dims must be positive, got {dims}")
    m_t = min(8, dims.m)
    n_t = min(8, dims.n)
    if dims.m <= 64:
        m_b = _round_up(dims.m, m_t)
    else:
        m_b = next((c for c in (64, 56, 48, 40, 32) if c % m_t == 0 and dims.m % c == 0), 64)
    n_b = _round_up(dims.n, n_t) if dims.n <= 128 else 128
    k_b = min(128, dims.k)
    return TilePlan(m_b=m_b, n_b=n_b, k_b=k_b, m_t=m_t, n_t=n_t)


# CTA tiles compiled into the FP32 CUDA-core kernel (csrc/conv_simt.cu), index = block_cfg.
# SIMT_TILES use 8x8 register micro-tiles (every TilePlan toggle compiled); SIMT_TILES_MT4
# (block_cfg 4..6) use 4x4 micro-tiles for layers too small to fill the GPU with 8x8 threads.
SIMT_TILES = ((128, 128), (64, 256), (96, 128), (128, 64))
SIMT_TILES_MT4 = ((64, 64), (128, 32), (32, 128))
SIMT_K_SLAB = 16
SIMT_MICRO_TILE = (8, 8)


def simt_tile_for(dims: GemmDims) -> int:
    """Library's shape-based tile choice (mirrors im2win_simt_pick in csrc/conv_simt.cu)."""
    slots = 148 * 2
    m96 = dims.m % 64 != 0 and dims.m % 96 == 0
    ctas = (dims.m // 96) * -(-dims.n // 128) if m96 else -(-dims.m // 64) * -(-dims.n // 256)
    # a partial last wave is split off to 4x4 tiles by the launcher; only a grid under one
    # wave that leaves the GPU under 75% busy runs on 4x4 tiles throughout
    if ctas < slots and ctas / slots < 0.75:
        return 6 if m96 else 4
    return 2 if m96 else 1


def gpu_plan(dims: GemmDims) -> TilePlan:
    """The TilePlan the GPU library runs for `dims` when no plan is given."""
    cfg = simt_tile_for(dims)
    if cfg >= len(SIMT_TILES):
        bm, bn = SIMT_TILES_MT4[cfg - len(SIMT_TILES)]
        return TilePlan(m_b=bm, n_b=bn, k_b=SIMT_K_SLAB, m_t=4, n_t=4)
    bm, bn = SIMT_TILES[cfg]
    return TilePlan(m_b=bm, n_b=bn, k_b=SIMT_K_SLAB, m_t=8, n_t=8)


def to_c_plan(plan: TilePlan | None):
    """Translate a TilePlan into the C ABI's im2win_tile_plan (None -> library default)."""
    from ._lib import TilePlanC

    if plan is None:
        return None
    cfg = -1
    if (plan.m_b, plan.n_b) in SIMT_TILES and plan.m_t == 8 and plan.n_t == 8:
        cfg = SIMT_TILES.index((plan.m_b, plan.n_b))
    elif (plan.m_b, plan.n_b) in SIMT_TILES_MT4 and plan.m_t == 4 and plan.n_t == 4:
        cfg = len(SIMT_TILES) + SIMT_TILES_MT4.index((plan.m_b, plan.n_b))
    return TilePlanC(cfg, int(plan.micro_kernel), int(plan.vectorized_load),
                     int(plan.prefetch_double_buffer))
