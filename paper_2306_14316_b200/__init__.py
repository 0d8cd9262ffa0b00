"""im2win convolution on B200 (sm_100a): a drop-in for the `winconv` im2win path.

Public names follow the reference package (/root/reference/pkg/src/winconv/__init__.py:47-86)
for the hot path: `im2win`, `Im2winTensor`, `conv_im2win_opt`,
`compute_from_windows_opt`, `TilePlan`, `default_plan`, `GemmDims`,
`ConvParams`, `Tensor4`, `output_dims`, `max_rel_diff`, `footprint_elems`,
`im2win_gather`, the error types and the benchmark harness (`run_bench`,
`run_ablation`, `search_plan`, `report_csv`, `footprint_report`, `BenchRecord`, `ALGORITHMS`).
The reference's CPU baselines (`conv_direct`, `conv_im2col_gemm`,
`conv_implicit_gemm`, `gemm`, `im2col`, `Mat2`) and its worker pool are not
rebuilt: on the GPU the baselines are cuDNN and im2col+cuBLAS (harness
algorithms "cudnn" / "im2col-cublas") and the CPU oracle lives in oracle/.  Operands live on CUDA devices; the
kernels are hand-written sm_100a CUDA in libim2win_sm100.so (csrc/), reached
through a C ABI (include/im2win_sm100.h).  There is no CPU fallback.
"""

from .errors import (
    FixtureFormatError,
    GeometryError,
    KernelError,
    MemoryBudgetError,
    PlanError,
    ShapeError,
    WinconvError,
)
from .tensors import ConvParams, Tensor4, check_conv_operands, max_rel_diff, normalized_max_diff, output_dims
from .plan import GemmDims, TilePlan, compose_k, compose_n, decompose_k, decompose_n, default_plan, gpu_plan
from .layouts import Im2winTensor, effective_width, footprint_elems, im2win, im2win_gather
from .kernels import (
    CapturedConv,
    compute_from_windows_basic,
    compute_from_windows_opt,
    conv_im2win_basic,
    conv_im2win_opt,
    conv_im2win_opt_host,
    conv_im2win_opt_host_batch,
)
from .workloads import BENCHMARKS, BenchConfig, make_inputs
from .fixture_io import read_tensor, write_tensor
from .harness import (
    ALGORITHMS,
    BenchRecord,
    footprint_report,
    report_csv,
    run_ablation,
    run_bench,
    search_plan,
)

__version__ = "0.1.0"

VARIANTS = ("fp32-exact", "fp32-fma", "tf32", "bf16")

__all__ = [
    "ALGORITHMS",
    "BenchRecord",
    "footprint_report",
    "report_csv",
    "run_ablation",
    "run_bench",
    "search_plan",
    "BENCHMARKS",
    "BenchConfig",
    "CapturedConv",
    "ConvParams",
    "FixtureFormatError",
    "GemmDims",
    "GeometryError",
    "Im2winTensor",
    "KernelError",
    "MemoryBudgetError",
    "PlanError",
    "ShapeError",
    "Tensor4",
    "TilePlan",
    "VARIANTS",
    "WinconvError",
    "check_conv_operands",
    "compose_k",
    "compose_n",
    "compute_from_windows_basic",
    "compute_from_windows_opt",
    "conv_im2win_basic",
    "conv_im2win_opt",
    "conv_im2win_opt_host",
    "conv_im2win_opt_host_batch",
    "decompose_k",
    "decompose_n",
    "default_plan",
    "effective_width",
    "footprint_elems",
    "gpu_plan",
    "im2win",
    "im2win_gather",
    "make_inputs",
    "max_rel_diff",
    "normalized_max_diff",
    "output_dims",
    "read_tensor",
    "write_tensor",
]
