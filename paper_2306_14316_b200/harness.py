"""GPU benchmark harness with the reference's record/CSV contract.

Mirrors winconv `bench.py` (/root/reference/pkg/src/winconv/bench.py): `ALGORITHMS`
(:32), `ABLATION_VARIANTS` (:37), `BenchRecord` (:112-145), `checksum_tensor`
(:148-149), `run_bench` (:226-266), `run_ablation` (:269-282), `report_csv`
(:297-308, same 17 leading columns + GPU columns) and `footprint_report`
(:321-331).  Protocol as in the reference (one warm-up, best of R repeats,
transform and compute timed separately, TFLOPS = flops / (transform + compute)),
timed with CUDA events on the current stream.  The memory-budget check uses the
device's free memory (the reference uses host RAM, bench.py:179-183).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, replace

import torch
import torch.nn.functional as F

from .errors import MemoryBudgetError
from .kernels import (
    basic_windows_into,
    conv_direct_into,
    conv_fused_into,
    conv_windows_into,
    direct_preferred,
    nhwc_into,
    nhwc_pitch,
)
from .layouts import im2win_into
from .plan import SIMT_K_SLAB, SIMT_TILES, SIMT_TILES_MT4, TilePlan, gpu_plan
from .workloads import BENCHMARKS, BenchConfig, make_inputs

ALGORITHMS = ("im2win-opt", "im2win-basic", "im2win-fma", "im2win-tf32", "im2win-bf16", "cudnn", "im2col-cublas")
ABLATION_VARIANTS = ("full", "-prefetch-double-buffer", "-vectorized-load", "-micro-kernel")
CSV_COLUMNS = ("name", "algorithm", "variant", "batch", "repeats", "h_o", "w_o",
               "flops", "transform_s", "compute_s", "total_s", "tflops",
               "raw_elems", "im2col_elems", "im2win_elems",
               "footprint_reduction_pct", "checksum",
               # GPU columns
               "device", "peak_mem_bytes", "timing_spread_s")
_MEM_SLACK = 1.1


@dataclass(frozen=True)
class BenchRecord:
    name: str
    algorithm: str
    variant: str
    batch: int
    repeats: int
    h_out: int
    w_out: int
    flops: int
    transform_s: float
    compute_s: float
    total_s: float
    tflops: float
    raw_elems: int
    im2col_elems: int
    im2win_elems: int
    footprint_reduction_pct: float
    checksum: str
    device: str = ""
    peak_mem_bytes: int = 0
    timing_spread_s: float = 0.0


def checksum_tensor(t: torch.Tensor) -> str:
    """sha256[:16] of the float32 bytes (bench.py:148-149)."""
    return hashlib.sha256(t.detach().contiguous().cpu().numpy().tobytes()).hexdigest()[:16]


def estimate_bytes(cfg: BenchConfig, algorithm: str) -> int:
    elems = cfg.elems("raw") + cfg.filter_elems + cfg.out_elems
    if algorithm == "im2col-cublas":
        elems += cfg.elems("im2col")
    elif algorithm in ("im2win-tf32", "im2win-bf16"):
        elems += cfg.elems("raw")
    else:
        elems += cfg.elems("im2win")
    return 4 * elems


def _check_memory_budget(cfg: BenchConfig, algorithm: str, device) -> None:
    required = int(estimate_bytes(cfg, algorithm) * _MEM_SLACK)
    free, _total = torch.cuda.mem_get_info(device)
    if required > free:
        raise MemoryBudgetError(required, free)


def _make_device_inputs(cfg: BenchConfig, device) -> tuple[torch.Tensor, torch.Tensor]:
    """The reference's seeded operands (numpy PCG64, bench.py:152-159) uploaded to the device,
    so a record's checksum equals the reference's record for the same config."""
    inp, flt = make_inputs(cfg)
    return torch.from_numpy(inp).to(device), torch.from_numpy(flt).to(device)


class _IeeeFp32:
    """True-FP32 PyTorch baselines: torch 2.11 runs cuDNN float32 convolutions in TF32 by default."""

    def __enter__(self):
        conv = getattr(torch.backends.cudnn, "conv", None)
        self._saved = (conv.fp32_precision, torch.backends.cuda.matmul.fp32_precision) if conv is not None else \
            (torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32)
        if conv is not None:
            conv.fp32_precision = "ieee"
            torch.backends.cuda.matmul.fp32_precision = "ieee"
        else:
            torch.backends.cudnn.allow_tf32 = torch.backends.cuda.matmul.allow_tf32 = False
        return self

    def __exit__(self, *exc):
        conv = getattr(torch.backends.cudnn, "conv", None)
        if conv is not None:
            conv.fp32_precision, torch.backends.cuda.matmul.fp32_precision = self._saved
        else:
            torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32 = self._saved
        return False


def _stages(cfg: BenchConfig, algorithm: str, x, f, plan: TilePlan | None):
    """(transform, compute, output) callables for one algorithm; buffers allocated once."""
    p = cfg.params
    h_out, w_out = cfg.out_dims
    out = torch.empty((cfg.batch, cfg.c_out, h_out, w_out), device=x.device)
    if algorithm in ("im2win-opt", "im2win-basic", "im2win-fma"):
        win = torch.empty((cfg.batch, cfg.c_in, h_out, cfg.h_f * cfg.w_eff), device=x.device)
        tr = lambda: im2win_into(x, win, p)  # noqa: E731
        if algorithm == "im2win-basic":
            cv = lambda: basic_windows_into(win, f, out, p)  # noqa: E731
        else:
            variant = "fp32-exact" if algorithm == "im2win-opt" else "fp32-fma"
            cv = lambda: conv_windows_into(win, f, out, p, cfg.w_eff, plan, variant)  # noqa: E731
        return tr, cv, out
    if algorithm in ("im2win-tf32", "im2win-bf16"):
        variant = algorithm[7:]
        if direct_preferred(x.shape, p, variant):  # the library's auto choice: in-SM windows from NCHW
            return (lambda: None), (lambda: conv_direct_into(x, f, out, p, variant)), out
        xc = torch.empty((cfg.batch, cfg.h_in + 2 * p.pad, cfg.w_in + 2 * p.pad, nhwc_pitch(cfg.c_in, variant)),
                         device=x.device, dtype=torch.bfloat16 if variant == "bf16" else torch.float32)
        return (lambda: nhwc_into(x, xc, p.pad)), (lambda: conv_fused_into(xc, f, out, p, variant)), out
    if algorithm == "cudnn":
        def cv():
            with _IeeeFp32():
                out.copy_(F.conv2d(x, f, stride=cfg.stride, padding=p.pad))
        return (lambda: None), cv, out
    if algorithm == "im2col-cublas":
        cols = {}

        def tr():
            cols["c"] = F.unfold(x, (cfg.h_f, cfg.w_f), stride=cfg.stride, padding=p.pad)

        def cv():
            with _IeeeFp32():
                torch.matmul(f.view(cfg.c_out, -1), cols["c"], out=out.view(cfg.batch, cfg.c_out, -1))
        return tr, cv, out
    raise ValueError(f"unknown algorithm {algorithm!r}, expected one of {ALGORITHMS}")


# The reference's CPU baselines (bench.py:32) map onto their GPU counterparts on this device:
# its per-image im2col + GEMM becomes im2col + cuBLAS, its direct and implicit-GEMM loops
# become cuDNN (which picks implicit GEMM / Winograd / FFT itself).
REFERENCE_ALIASES = {"im2col-gemm": "im2col-cublas", "direct": "cudnn", "implicit-gemm": "cudnn"}


def run_bench(cfg: BenchConfig, variant: str = "-", *, device=None) -> BenchRecord:
    """Warm up once, run `cfg.repeats` times, report the fastest run (bench.py:226-266).

    Same call as the reference: `cfg.algorithm`, `cfg.repeats` and `cfg.plan` come from
    the config (bench.py:43-59), `variant` is the record's label.  Extras are keyword-only.
    """
    algorithm = REFERENCE_ALIASES.get(cfg.algorithm, cfg.algorithm)
    if algorithm not in ALGORITHMS:
        raise ValueError(f"unknown algorithm {cfg.algorithm!r}, expected one of {ALGORITHMS}")
    if cfg.repeats < 1:
        raise ValueError("repeats must be >= 1")
    repeats, plan = cfg.repeats, cfg.plan
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    _check_memory_budget(cfg, algorithm, dev)
    prev_tf32 = torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32
    torch.backends.cudnn.allow_tf32 = torch.backends.cuda.matmul.allow_tf32 = False
    try:
        with torch.cuda.device(dev):
            x, f = _make_device_inputs(cfg, dev)
            torch.cuda.synchronize(dev)
            base = torch.cuda.memory_allocated(dev)
            torch.cuda.reset_peak_memory_stats(dev)
            tr, cv, out = _stages(cfg, algorithm, x, f, plan)
            tr()
            cv()
            torch.cuda.synchronize(dev)
            peak = torch.cuda.max_memory_allocated(dev) - base
            stream = torch.cuda.current_stream(dev)
            best, totals = None, []
            for _ in range(repeats):
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                e[0].record(stream)
                tr()
                e[1].record(stream)
                cv()
                e[2].record(stream)
                torch.cuda.synchronize(dev)
                t_tr, t_cv = e[0].elapsed_time(e[1]) * 1e-3, e[1].elapsed_time(e[2]) * 1e-3
                totals.append(t_tr + t_cv)
                if best is None or totals[-1] < best[0]:
                    best = (totals[-1], t_tr, t_cv)
            checksum = checksum_tensor(out)
    finally:
        torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32 = prev_tf32
    total, t_tr, t_cv = best
    h_out, w_out = cfg.out_dims
    col, win = cfg.elems("im2col"), cfg.elems("im2win")
    return BenchRecord(
        name=cfg.name, algorithm=cfg.algorithm, variant=variant, batch=cfg.batch, repeats=repeats, h_out=h_out,
        w_out=w_out, flops=cfg.flops, transform_s=t_tr, compute_s=t_cv, total_s=total,
        tflops=cfg.flops / total / 1e12, raw_elems=cfg.elems("raw"), im2col_elems=col, im2win_elems=win,
        footprint_reduction_pct=100.0 * (1.0 - win / col), checksum=checksum, device=torch.cuda.get_device_name(dev),
        peak_mem_bytes=int(peak), timing_spread_s=max(totals) - min(totals))


def run_ablation(cfg: BenchConfig, *, device=None) -> list[BenchRecord]:
    """Full tiled kernel, then each optimisation removed one at a time (bench.py:269-282, paper Fig. 4).

    The base plan is `cfg.plan` when given, else the tile the GPU library runs for the shape.
    """
    base = cfg.plan if cfg.plan is not None else gpu_plan(cfg.gemm_dims())
    plans = {
        "full": base,
        "-prefetch-double-buffer": base.with_toggles(prefetch_double_buffer=False),
        "-vectorized-load": base.with_toggles(vectorized_load=False),
        "-micro-kernel": base.with_toggles(micro_kernel=False),
    }
    return [run_bench(replace(cfg, algorithm="im2win-opt", plan=plan), label, device=device)
            for label, plan in plans.items()]


# The reference searches (m_b, n_b, k_b) over a CPU grid (bench.py:334-339).  On the GPU the
# searchable space is the set of CTA tiles compiled into the FP32 kernel (plan.SIMT_TILES*),
# each with its own register micro-tile and the 16-deep K slab.
DEFAULT_SEARCH_GRID = tuple((m_b, n_b, SIMT_K_SLAB) for m_b, n_b in SIMT_TILES + SIMT_TILES_MT4)


def _compiled_plan(m_b: int, n_b: int, k_b: int) -> TilePlan | None:
    if k_b != SIMT_K_SLAB:
        return None
    if (m_b, n_b) in SIMT_TILES:
        return TilePlan(m_b=m_b, n_b=n_b, k_b=k_b, m_t=8, n_t=8)
    if (m_b, n_b) in SIMT_TILES_MT4:
        return TilePlan(m_b=m_b, n_b=n_b, k_b=k_b, m_t=4, n_t=4)
    return None


def search_plan(cfg: BenchConfig, grid=DEFAULT_SEARCH_GRID, repeats: int = 1, *,
                device=None) -> list[tuple[TilePlan, float]]:
    """Grid search over block extents; returns (plan, seconds) sorted fastest-first (bench.py:342-364).

    Grid entries that do not name a compiled GPU tile are skipped, as the reference skips
    entries whose micro-tile does not divide the block.  Each plan is warmed up once and
    timed `repeats` times with CUDA events on the current stream (best run kept).
    """
    if repeats < 1:
        raise ValueError("repeats must be >= 1")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    p = cfg.params
    results = []
    with torch.cuda.device(dev):
        x, f = _make_device_inputs(cfg, dev)
        h_out, w_out = cfg.out_dims
        win = torch.empty((cfg.batch, cfg.c_in, h_out, cfg.h_f * cfg.w_eff), device=dev)
        out = torch.empty((cfg.batch, cfg.c_out, h_out, w_out), device=dev)
        im2win_into(x, win, p)
        stream = torch.cuda.current_stream(dev)
        seen = set()
        for m_b, n_b, k_b in grid:
            plan = _compiled_plan(m_b, n_b, k_b)
            if plan is None or plan in seen:
                continue
            seen.add(plan)
            conv_windows_into(win, f, out, p, cfg.w_eff, plan)  # warm-up
            best = float("inf")
            for _ in range(repeats):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                conv_windows_into(win, f, out, p, cfg.w_eff, plan)
                b.record(stream)
                torch.cuda.synchronize(dev)
                best = min(best, a.elapsed_time(b) * 1e-3)
            results.append((plan, best))
    results.sort(key=lambda pair: pair[1])
    return results


def _fmt(value) -> str:
    if isinstance(value, float):
        return f"{value:.6g}"
    return str(value)


def report_csv(records: list[BenchRecord]) -> str:
    """Render records as CSV ordered by (config, algorithm, variant) (bench.py:297-308)."""
    if not records:
        raise ValueError("no records to report")
    order = list(BENCHMARKS)

    def key(r):
        return (order.index(r.name) if r.name in order else len(order), r.name, r.algorithm, r.variant)

    lines = [",".join(CSV_COLUMNS)]
    for r in sorted(records, key=key):
        row = (r.name, r.algorithm, r.variant, r.batch, r.repeats, r.h_out, r.w_out, r.flops, r.transform_s,
               r.compute_s, r.total_s, r.tflops, r.raw_elems, r.im2col_elems, r.im2win_elems,
               r.footprint_reduction_pct, r.checksum, r.device, r.peak_mem_bytes, r.timing_spread_s)
        lines.append(",".join(_fmt(v) for v in row))
    return "\n".join(lines) + "\n"


@dataclass(frozen=True)
class FootprintRow:
    name: str
    batch: int
    raw_elems: int
    im2col_elems: int
    im2win_elems: int
    reduction_pct: float


def footprint_report(cfgs: list[BenchConfig]) -> list[FootprintRow]:
    """Per-config element counts per layout plus the window-vs-column saving (bench.py:321-331)."""
    rows = []
    for cfg in cfgs:
        col, win = cfg.elems("im2col"), cfg.elems("im2win")
        rows.append(FootprintRow(cfg.name, cfg.batch, cfg.elems("raw"), col, win, 100.0 * (1.0 - win / col)))
    return rows


def layer_configs(batch: int) -> list[BenchConfig]:
    return [replace(c, batch=batch, seed=1000 + i) for i, c in enumerate(BENCHMARKS.values())]
