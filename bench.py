#!/usr/bin/env python
"""Benchmark: im2win transform + convolution over the paper's 12 layers on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--variant fp32-exact|fp32-fma|tf32|bf16] [--detail PATH]

A *step* is one pass of the hot path (im2win transform + im2win convolution)
over all twelve benchmark layers (BASELINE.json configs[1]:
/root/reference/pkg/src/winconv/bench.py:88-104) at N=128 images per GPU; the
default variant is the FP32-exact kernel (bit-identical to the reference).
`value` = total algorithmic FLOPs of all ranks / max-over-ranks device time
(TFLOPS, FLOPs = 2*N*Co*Ho*Wo*Ci*Hf*Wf as in winconv bench.py:70-74; the
transform is inside the timed region, as in the reference's TFLOPS, bench.py:259).
Multi-GPU is batch sharding (weak scaling: each rank owns its own 128-image
slice), no collective on the data path.

Besides the headline step every rank runs the tensor-core legs of the other
BASELINE configs through the production TF32/BF16 path: config 4 (conv9-12 at a
global N=1024 split over the ranks) and config 5 (all 12 layers at a global
N=2048 split over the ranks), each layer timed as the max over ranks with a
per-layer roofline fraction.  Rank 0 adds cuDNN / im2col+cuBLAS baselines, the
memory footprints and the CPU oracle.  stdout gets ONE compact JSON line (< 2 KB)
as the last line; every per-layer table goes to the `--detail` sidecar file.

`--gpus N` without a launcher re-executes itself under torch.distributed.run
with N ranks (NCCL, one GPU per rank; gloo when ranks must share a GPU).

`--impl reference` times the CPU oracle (a C restatement of the reference's
algorithm, oracle/) on a bounded sample of the same workload on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from dataclasses import replace
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "TFLOPS per conv layer (12 benchmarks) at 1/2/4/8 B200; memory footprint"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}
LINE_LIMIT = 2000


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return dict(PEAKS_FALLBACK)


def pinned(t):
    """Page-locked copy of a host tensor; pageable if the host cannot pin that much (the
    streamed host path still works, its copies just stop overlapping)."""
    try:
        return t.pin_memory()
    except RuntimeError:
        return t


def max_rel_diff_device(a, b) -> float:
    """winconv max_rel_diff (tensors.py:135-150) evaluated on the GPU: identical bits -> 0."""
    import torch

    a64, b64 = a.double(), b.double()
    d = (a64 - b64).abs() / torch.clamp(torch.maximum(a64.abs(), b64.abs()), min=1.0)
    d[a.view(torch.int32) == b.view(torch.int32)] = 0
    return float(d.max().item())


def set_fp32_precision(mode: str) -> None:
    """Float32 conv/matmul precision of the PyTorch baselines: "ieee" (true FP32) or "tf32".

    torch 2.11 defaults cuDNN convolutions to TF32 (torch.backends.cudnn.conv.fp32_precision
    == "tf32"); allow_tf32 = False alone leaves that default in place.
    """
    import torch

    conv = getattr(torch.backends.cudnn, "conv", None)
    if conv is not None and hasattr(conv, "fp32_precision"):
        conv.fp32_precision = mode
        torch.backends.cuda.matmul.fp32_precision = mode
    else:
        torch.backends.cudnn.allow_tf32 = mode == "tf32"
        torch.backends.cuda.matmul.allow_tf32 = mode == "tf32"


def pcie_probe(dev, stream, nbytes: int = 256 << 20) -> dict:
    """Pinned host<->device copy bandwidth (GB/s): H2D alone, D2H alone, both at once."""
    import torch

    hs = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    hd = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    da = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    db = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    side = torch.cuda.Stream(dev)

    def timed(fn):
        fn()
        best = 1e30
        for _ in range(3):
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            best = min(best, e0.elapsed_time(e1) * 1e-3)
        return nbytes / best / 1e9

    def both():
        side.wait_stream(stream)
        da.copy_(hs, non_blocking=True)
        with torch.cuda.stream(side):
            hd.copy_(db, non_blocking=True)
        stream.wait_stream(side)

    return {"h2d_gbs": timed(lambda: da.copy_(hs, non_blocking=True)),
            "d2h_gbs": timed(lambda: hd.copy_(db, non_blocking=True)), "bidir_each_gbs": timed(both)}


def load_traffic(names, batch: int, variant: str, path: str = "windows"):
    """DRAM traffic of the step's conv kernels from a committed ncu capture.

    path "windows" (conv over Ĩ): profiles/r01_traffic_n128.json, tools/ncu_traffic.py (one
    `ncu --set full` capture per layer); path "nchw" (windows gathered from NCHW):
    profiles/r02_traffic_nchw_n128.json, tools/ncu_traffic_nchw.py.  dram__bytes_read.sum +
    dram__bytes_write.sum per conv call.  Returns None when no capture covers this workload.
    """
    for p in sorted((ROOT / "profiles").glob("r*_traffic*_n128.json"), reverse=True):
        d = json.loads(p.read_text())
        if (d.get("batch") != batch or d.get("variant") != variant or d.get("path", "windows") != path
                or not all(n in d["layers"] for n in names)):
            continue
        conv = [d["layers"][n]["conv_dram_bytes"] for n in names]
        alg = [d["layers"][n]["conv_algorithmic_bytes"] for n in names]
        out = {"source": str(p.relative_to(ROOT)), "capture": d.get("capture"),
               "conv_bytes_per_launch": sum(conv) / len(conv),
               "per_launch_note": "per layer conv call (mean over the 12 layers); a tail-split layer's two "
                                  "kernel launches count as one call",
               "conv_algorithmic_bytes_per_launch": sum(alg) / len(alg),
               "per_layer": {n: d["layers"][n] for n in names}}
        if all("transform_dram_bytes" in d["layers"][n] for n in names):
            out["transform_bytes_per_launch"] = sum(d["layers"][n]["transform_dram_bytes"] for n in names) / len(names)
        return out
    return None


def load_tc_traffic(variant: str):
    """Per-layer DRAM bytes of the production TC path (tools/ncu_traffic_tc.py capture), or None."""
    for p in sorted((ROOT / "profiles").glob(f"r*_tc_traffic_{variant}_n128.json"), reverse=True):
        d = json.loads(p.read_text())
        return {"source": str(p.relative_to(ROOT)), "layers": d["layers"]}
    return None


# ---------------------------------------------------------------------------
# reference arm: CPU oracle on the host cores
# ---------------------------------------------------------------------------
def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as orc
    from paper_2306_14316_b200.workloads import BENCHMARKS, make_inputs

    threads = orc.max_threads()
    sample_batch = 1
    cfgs = [replace(c, batch=sample_batch, seed=i) for i, c in enumerate(BENCHMARKS.values())]
    ops = [make_inputs(c) for c in cfgs]
    flops = sum(c.flops for c in cfgs)

    def step():
        for c, (inp, flt) in zip(cfgs, ops):
            win = orc.im2win_fill(inp, c.h_f, c.w_f, c.stride, threads)
            orc.conv_from_windows(win, flt, c.stride, c.out_dims[1], threads)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    value = flops / dt / 1e12
    sample = "12 layers at N=1 image per step (per-image slice of the N=128 workload), transform + unfused-f32 conv"
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "TFLOPS", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic N(0,1), numpy PCG64 seeded",
        "config": {"workload": "paper 12 conv layers, im2win transform + conv (CPU oracle port, bounded sample)",
                   "per_step_batch": sample_batch, "parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": value, "unit": "TFLOPS", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks sampler
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.device_index = device_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device_index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self._t.join(timeout=2)
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
                pw.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if s > 0.5 * (max(mx) if mx else 0)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(n: int) -> None:
    """`bench.py --gpus N` with no launcher: re-exec as N ranks of one node (never returns)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    print(f"[bench] launching {n} ranks: {' '.join(cmd[1:])}", file=sys.stderr, flush=True)
    os.execv(sys.executable, cmd)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
class Dist:
    """Rank plumbing: one process per GPU, barrier + max over ranks for every timed number."""

    def __init__(self):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        n_dev = torch.cuda.device_count()
        # NCCL needs one GPU per rank; ranks sharing a GPU (tests on a 1-GPU box) use gloo
        default = "nccl" if n_dev >= self.world else "gloo"
        self.backend = os.environ.get("IM2WIN_DIST_BACKEND", default)
        self.dev = torch.device("cuda", local_rank % n_dev if self.world > 1 else 0)
        torch.cuda.set_device(self.dev)
        if self.world > 1:
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group(self.backend)
        props = torch.cuda.get_device_properties(self.dev)
        uuid = str(getattr(props, "uuid", self.dev.index))
        uuids = [uuid]
        if self.world > 1:
            uuids = [None] * self.world
            dist.all_gather_object(uuids, uuid)
        self.devices_distinct = len(set(uuids))
        print(f"[bench] rank {self.rank}/{self.world} backend={self.backend if self.world > 1 else 'none'} "
              f"device={self.dev} {props.name} uuid={uuid}", file=sys.stderr, flush=True)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device=self.dev if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.barrier()
            self.dist.destroy_process_group()


def tensor_peaks(dev, stream) -> dict:
    """Dense tensor-core peaks measured here with cuBLAS (8192^3 GEMMs, best of 10): bf16 and tf32."""
    import torch

    out = {}
    n = 8192
    for name, dt, prec in (("bf16", torch.bfloat16, "ieee"), ("tf32", torch.float32, "tf32")):
        set_fp32_precision(prec)
        a = torch.randn((n, n), device=dev, dtype=dt)
        b = torch.randn((n, n), device=dev, dtype=dt)
        c = torch.matmul(a, b)
        best = 1e30
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            torch.matmul(a, b, out=c)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            best = min(best, e0.elapsed_time(e1) * 1e-3)
        out[name] = 2 * n ** 3 / best / 1e12
        del a, b, c
    set_fp32_precision("ieee")
    torch.cuda.empty_cache()
    return out


def fp32_peaks(lib, dev, stream) -> dict:
    """FP32 CUDA-core peaks measured in this run: the bit-exact multiply-then-add as scalar FMUL+FADD
    and in the packed FFMA2 form the conv kernel issues (`exact` = the higher of the two: the ceiling
    of a bit-exact conv), and FFMA chains."""
    import torch

    sink = torch.empty(256, device=dev)
    peak = {}
    for mode, key, chains in ((1, "exact_scalar", 32), (2, "exact_packed", 64), (0, "ffma", 32)):
        iters, blocks = 1 << 15, 148 * 8
        lib.im2win_bench_fp32_peak(sink.data_ptr(), mode, 256, blocks, stream.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        lib.im2win_bench_fp32_peak(sink.data_ptr(), mode, iters, blocks, stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        peak[key] = 2 * chains * iters * 256 * blocks / (e0.elapsed_time(e1) * 1e-3) / 1e12
    peak["exact"] = max(peak["exact_scalar"], peak["exact_packed"])
    return peak


def tc_min_bytes(cfg, variant: str) -> int:
    """Algorithmic HBM bytes of one TC layer call: read the NCHW f32 input and the filter once,
    write the NCHW f32 output once (whatever intermediate the path makes is overhead)."""
    return 4 * (cfg.elems("raw") + cfg.filter_elems + cfg.out_elems)


def roofline_row(flops: float, nbytes: float, seconds: float, peak_tf: float, hbm_gbs: float) -> dict:
    """min(tensor peak, AI x HBM) bound for one layer and the fraction reached."""
    t_compute = flops / (peak_tf * 1e12)
    t_mem = nbytes / (hbm_gbs * 1e9)
    bound = "tensor" if t_compute >= t_mem else "hbm"
    attainable = flops / max(t_compute, t_mem) / 1e12
    achieved = flops / seconds / 1e12
    return {"bound": bound, "attainable_tflops": attainable, "achieved_tflops": achieved,
            "frac": achieved / attainable, "alg_bytes": nbytes}


def _feed_chosen(cfg, variant: str) -> bool:
    """Mirror of the library's feed rule (conv_tc_fused.cu): the channels-last copy is produced
    inside the conv kernel when output/input elements <= 0.5 and N <= 256, or when IM2WIN_FEED=2."""
    mode = os.environ.get("IM2WIN_FEED", "1")
    h_out, w_out = cfg.out_dims
    r = cfg.c_out * h_out * w_out / (cfg.c_in * cfg.h_in * cfg.w_in)
    return mode == "2" or (mode == "1" and r <= 0.5 and cfg.batch <= 256)


def tc_layer(D, cfg_global, variant: str, reps: int = 5) -> dict:
    """Time the production TF32/BF16 path for one layer at a global batch split over the ranks.

    Each rank transforms and convolves its contiguous slice (sharding.shard_bounds); the
    launch sequence is captured in CUDA graphs (transform+conv, and conv alone) and replayed
    `reps` times between events after a barrier; the time is the max over ranks.
    """
    import torch

    from paper_2306_14316_b200 import _lib
    from paper_2306_14316_b200.kernels import (
        conv_direct_into,
        conv_fused_into,
        conv_fused_nchw_into,
        direct_preferred,
        nhwc_pitch,
    )
    from paper_2306_14316_b200.sharding import shard_bounds

    dev = D.dev
    stream = torch.cuda.current_stream(dev)
    lo, hi = shard_bounds(cfg_global.batch, D.world, D.rank)
    cfg = replace(cfg_global, batch=hi - lo)
    h_out, w_out = cfg.out_dims
    g = torch.Generator(device=dev).manual_seed(cfg.seed + 7919 * D.rank)
    x = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev, generator=g)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev, generator=g)
    torch.cuda.synchronize(dev)
    base = torch.cuda.memory_allocated(dev)
    torch.cuda.reset_peak_memory_stats(dev)
    o = torch.empty((cfg.batch, cfg.c_out, h_out, w_out), device=dev)
    lib = _lib.load()
    code = _lib.VARIANTS[variant]
    if direct_preferred(x.shape, cfg.params, variant):
        ws = torch.empty(max(lib.im2win_conv_direct_workspace(cfg.c_in, cfg.c_out, cfg.h_f, cfg.w_f, code), 1 << 16),
                         dtype=torch.uint8, device=dev)
        one = None
        cv = lambda: conv_direct_into(x, f, o, cfg.params, variant, ws)  # noqa: E731
        cv()
        path = _lib.last_kernel()
    else:
        # production: one call (im2win_conv_fused_nchw) -- the library produces the channels-last
        # copy inside the conv kernel (feed) or with its copy kernel just before it; "conv" times
        # the conv kernel alone on an existing copy
        ws = torch.empty(max(lib.im2win_conv_fused_nchw_workspace_bytes(cfg.batch, cfg.c_in, cfg.c_out, cfg.h_f,
                                                                        cfg.w_f), 1 << 16),
                         dtype=torch.uint8, device=dev)
        w = torch.empty((cfg.batch, cfg.h_in, cfg.w_in, nhwc_pitch(cfg.c_in, variant)),
                        dtype=torch.bfloat16 if variant == "bf16" else torch.float32, device=dev)
        one = lambda: conv_fused_nchw_into(x, w, f, o, cfg.params, variant, ws)  # noqa: E731
        cv = lambda: conv_fused_into(w, f, o, cfg.params, variant, ws)  # noqa: E731
        one()
        path = "one call (" + ("in-kernel NHWC feed" if _feed_chosen(cfg, variant) else "NHWC copy kernel") + ") + " \
            + _lib.last_kernel()
        cv()
    torch.cuda.synchronize(dev)
    peak_mem = torch.cuda.max_memory_allocated(dev) - base

    def capture(fns):
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            for fn in fns:
                fn()
        stream.wait_stream(side)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, capture_error_mode="relaxed"):
            for fn in fns:
                fn()
        return gr

    g_all = capture([one] if one is not None else [cv])
    g_cv = capture([cv])
    times = {}
    for key, gr in (("all", g_all), ("conv", g_cv)):
        gr.replay()
        torch.cuda.synchronize(dev)
        D.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            gr.replay()
        b.record(stream)
        torch.cuda.synchronize(dev)
        times[key] = D.max(a.elapsed_time(b) / reps) * 1e-3
    del g_all, g_cv, x, f, o, ws
    torch.cuda.empty_cache()
    return {"s": times["all"], "conv_s": times["conv"], "path": path, "peak_mem_bytes_rank": peak_mem,
            "per_rank_batch": cfg.batch}


def windows_path_step(layers, variant: str, dev, stream, peaks, fp, D, reps: int = 5) -> dict:
    """The reference's two-call form -- im2win transform, then the tiled conv over Ĩ
    (layouts.py:86-95 + optimized.py:217-234) -- timed per layer after the headline region:
    the transform's HBM GB/s against the roofline, and the step this form would give."""
    import torch

    from paper_2306_14316_b200.kernels import conv_windows_into
    from paper_2306_14316_b200.layouts import im2win_into

    rows, tot_f, tot_s = {}, 0.0, 0.0
    for L in layers:
        cfg = L["cfg"]
        h_out, _ = cfg.out_dims
        mid = torch.empty((cfg.batch, cfg.c_in, h_out, cfg.h_f * cfg.w_eff), device=dev)
        tr = lambda: im2win_into(L["x"], mid, cfg.params)  # noqa: E731
        cv = lambda: conv_windows_into(mid, L["f"], L["out"], cfg.params, cfg.w_eff, None, variant)  # noqa: E731
        tr()
        cv()
        torch.cuda.synchronize(dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3 * reps)]
        for r in range(reps):
            ev[3 * r].record(stream)
            tr()
            ev[3 * r + 1].record(stream)
            cv()
            ev[3 * r + 2].record(stream)
        torch.cuda.synchronize(dev)
        t_tr = D.max(statistics.fmean(ev[3 * r].elapsed_time(ev[3 * r + 1]) for r in range(reps)))
        t_cv = D.max(statistics.fmean(ev[3 * r + 1].elapsed_time(ev[3 * r + 2]) for r in range(reps)))
        gbs = cfg.transform_bytes() / (t_tr * 1e-3) / 1e9
        rows[L["name"]] = {"transform_ms": t_tr, "transform_gbs": gbs, "transform_frac_of_hbm": gbs / peaks["hbm_gbs"],
                           "conv_ms": t_cv, "tflops": cfg.flops / ((t_tr + t_cv) * 1e-3) / 1e12,
                           "tflops_conv_only": cfg.flops / (t_cv * 1e-3) / 1e12}
        tot_f += cfg.flops
        tot_s += (t_tr + t_cv) * 1e-3
        del mid
    torch.cuda.empty_cache()
    return {"note": "im2win transform (TMA bulk copies) + conv over the materialised Ĩ, per layer, CUDA events, "
                    f"mean of {reps} after a warm-up, max over ranks; same bits as the headline path",
            "tflops_per_gpu": tot_f / tot_s / 1e12, "layers": rows}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=128, help="images per GPU in the headline step")
    ap.add_argument("--variant", default="fp32-exact", choices=["fp32-exact", "fp32-fma", "tf32", "bf16"])
    ap.add_argument("--layers", default="all")
    ap.add_argument("--no-baselines", action="store_true", help="skip cuDNN / im2col+cuBLAS / CPU legs")
    ap.add_argument("--no-tc", action="store_true", help="skip the TF32/BF16 config-4/5 legs")
    ap.add_argument("--windows-path", action="store_true",
                    help="headline FP32 step as transform + conv over Ĩ instead of the production NCHW-direct call")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--detail", default="gpurun_out/bench_detail.json", help="sidecar file with every table")
    args = ap.parse_args()

    if args.impl == "reference":
        run_reference(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch_under_torchrun(args.gpus)

    import torch

    import paper_2306_14316_b200 as pkg
    from paper_2306_14316_b200 import _lib
    from paper_2306_14316_b200.kernels import (
        conv_direct_into,
        conv_fused_into,
        conv_fused_nchw_into,
        conv_nchw_into,
        conv_windows_into,
        direct_preferred,
        nchw_direct,
        nhwc_into,
        nhwc_pitch,
    )
    from paper_2306_14316_b200.layouts import im2win_into
    from paper_2306_14316_b200.workloads import BENCHMARKS

    D = Dist()
    dev, rank, world = D.dev, D.rank, D.world
    set_fp32_precision("ieee")
    lib = _lib.load()
    names = list(BENCHMARKS) if args.layers == "all" else args.layers.split(",")
    peaks = load_peaks()
    tc_step = args.variant in ("tf32", "bf16")
    stream = torch.cuda.current_stream(dev)

    # ---- the headline step's operands, allocated once (inputs resident in HBM) ----
    gen = torch.Generator(device=dev)
    layers = []
    for i, name in enumerate(names):
        cfg = replace(BENCHMARKS[name], batch=args.batch, seed=1000 + i + 97 * rank)
        gen.manual_seed(cfg.seed)
        h_out, w_out = cfg.out_dims
        L = dict(name=name, cfg=cfg)
        L["x"] = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev, generator=gen)
        L["f"] = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev, generator=gen)
        L["out"] = torch.empty((cfg.batch, cfg.c_out, h_out, w_out), device=dev)
        if not tc_step and nchw_direct(cfg.params) and not args.windows_path:
            # production conv_im2win_opt: the tiled kernel gathers the im2win windows straight from
            # NCHW (im2win_conv_nchw_f32; no Ĩ pass, same bits); the transform + conv over Ĩ (the
            # compute_from_windows_opt seam) is timed after the headline region (detail.windows_path)
            L["tr"] = lambda: None
            L["cv"] = (lambda L=L: conv_nchw_into(L["x"], L["f"], L["out"], L["cfg"].params, None, args.variant))
        elif not tc_step:
            L["mid"] = torch.empty((cfg.batch, cfg.c_in, h_out, cfg.h_f * cfg.w_eff), device=dev)
            L["tr"] = (lambda L=L: im2win_into(L["x"], L["mid"], L["cfg"].params))
            L["cv"] = (lambda L=L: conv_windows_into(L["mid"], L["f"], L["out"], L["cfg"].params, L["cfg"].w_eff,
                                                     None, args.variant))
        elif direct_preferred(L["x"].shape, cfg.params, args.variant):
            L["tr"] = lambda: None
            L["cv"] = (lambda L=L: conv_direct_into(L["x"], L["f"], L["out"], L["cfg"].params, args.variant))
        else:
            L["mid"] = torch.empty((cfg.batch, cfg.h_in, cfg.w_in, nhwc_pitch(cfg.c_in, args.variant)), device=dev,
                                   dtype=torch.bfloat16 if args.variant == "bf16" else torch.float32)
            if cfg.params.pad:
                L["tr"] = (lambda L=L: nhwc_into(L["x"], L["mid"]))
                L["cv"] = (lambda L=L: conv_fused_into(L["mid"], L["f"], L["out"], L["cfg"].params, args.variant))
            else:  # production one-call path: the channels-last copy is part of the conv call
                L["tr"] = lambda: None
                L["cv"] = (lambda L=L: conv_fused_nchw_into(L["x"], L["mid"], L["f"], L["out"], L["cfg"].params,
                                                            args.variant))
        layers.append(L)

    def step():
        for L in layers:
            L["tr"]()
            L["cv"]()

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize(dev)
    kernel_of = {}
    for L in layers:
        L["cv"]()
        kernel_of[L["name"]] = _lib.last_kernel()

    # ---- timed region: exactly K steps ----
    # Events around every transform and conv call are recorded inside the timed region (same
    # stream, GPU kept busy by the queue) so the dominant kernel's average launch duration
    # comes from the run that produces `value`.
    n_l = len(layers)
    marks = [[[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n_l)]
             for _ in range(args.steps)]
    sampler = ClockSampler(dev.index)
    sampler.start()
    time.sleep(0.3)
    launches0 = lib.im2win_conv_launch_count()
    torch.cuda.synchronize(dev)
    D.barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for k in range(args.steps):
        for L, m in zip(layers, marks[k]):
            m[0].record(stream)
            L["tr"]()
            m[1].record(stream)
            L["cv"]()
            m[2].record(stream)
    ev1.record(stream)
    conv_launches = lib.im2win_conv_launch_count() - launches0
    torch.cuda.synchronize(dev)
    D.barrier()
    clocks = sampler.stop()
    elapsed_ms = D.max(ev0.elapsed_time(ev1))
    flops_step = sum(L["cfg"].flops for L in layers)
    value = flops_step * world * args.steps / (elapsed_ms * 1e-3) / 1e12
    ms_per_step = elapsed_ms / args.steps
    # transform (or channels-last copy) launches + the packed-filter launch of each conv call
    xform_launches = sum(1 for L in layers if "mid" in L) * args.steps
    gpu_launches = conv_launches + xform_launches + (n_l * args.steps if not tc_step else 0)

    # ---- per-layer breakdown from the timed region (mean over the K steps) ----
    fp = fp32_peaks(lib, dev, stream)
    per_layer = {}
    conv_ms_total = tr_ms_total = 0.0
    for li, L in enumerate(layers):
        cfg = L["cfg"]
        t_tr = statistics.fmean(marks[k][li][0].elapsed_time(marks[k][li][1]) for k in range(args.steps))
        t_cv = statistics.fmean(marks[k][li][1].elapsed_time(marks[k][li][2]) for k in range(args.steps))
        conv_ms_total += t_cv
        tr_ms_total += t_tr
        rec = {"transform_ms": t_tr, "conv_ms": t_cv, "tflops": cfg.flops / ((t_tr + t_cv) * 1e-3) / 1e12,
               "tflops_conv_only": cfg.flops / (t_cv * 1e-3) / 1e12, "kernel": kernel_of[L["name"]]}
        if not tc_step:
            pk = fp["exact"] if args.variant == "fp32-exact" else fp["ffma"]
            rec["roofline"] = {"bound": "fp32-simt", "peak_tflops": pk, "frac": rec["tflops_conv_only"] / pk}
            if "mid" in L:
                rec["transform_gbs"] = cfg.transform_bytes() / (t_tr * 1e-3) / 1e9
                rec["roofline"]["transform_frac_of_hbm"] = rec["transform_gbs"] / peaks["hbm_gbs"]
            else:
                rec["path"] = "windows gathered from NCHW (im2win_conv_nchw_f32), no transform pass"
        per_layer[L["name"]] = rec

    windows_path = None
    if not tc_step and not any("mid" in L for L in layers):
        windows_path = windows_path_step(layers, args.variant, dev, stream, peaks, fp, D)

    detail = {"metric": METRIC, "n_gpus": world, "devices_distinct": D.devices_distinct, "backend": D.backend,
              "headline_step": {"variant": args.variant, "per_gpu_batch": args.batch, "value_tflops": value,
                                "ms_per_step": ms_per_step, "layers": per_layer,
                                "path": "conv_im2win_opt production path" + (
                                    " (FP32: im2win windows gathered straight from NCHW, no Ĩ pass)"
                                    if windows_path is not None else "")},
              "windows_path": windows_path,
              "peaks": {"fp32_exact_tflops": fp["exact"], "fp32_exact_scalar_tflops": fp["exact_scalar"],
                        "fp32_exact_packed_tflops": fp["exact_packed"], "fp32_ffma_tflops": fp["ffma"],
                        "hbm_gbs": peaks["hbm_gbs"], "bf16_tflops_file": peaks.get("bf16_tflops"),
                        "source": peaks["source"] + "; fp32 probes measured in this run"}}

    # ---- e2e: public host API (numpy-style call: host operands in, host result out) ----
    # conv_im2win_opt_host streams each layer's batch in chunks (upload / transform+conv /
    # download overlapped on three streams, csrc/pipeline.cu); every byte crosses PCIe inside
    # the timed region.
    host = []
    for L in layers:
        host.append(dict(x=pinned(L["x"].cpu()), f=pinned(L["f"].cpu()),
                         out=pinned(torch.empty(L["out"].shape, dtype=torch.float32))))
    h2d = sum(h["x"].numel() * 4 + h["f"].numel() * 4 for h in host)
    d2h = sum(h["out"].numel() * 4 for h in host)

    def e2e_step():
        pkg.conv_im2win_opt_host_batch([(h["x"], h["f"], L["cfg"].params) for L, h in zip(layers, host)],
                                       variant=args.variant, outs=[h["out"] for h in host])

    e2e_step()
    torch.cuda.synchronize(dev)
    D.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = D.max(e0.elapsed_time(e1)) / args.e2e_steps
    if args.variant == "fp32-exact":
        e2e_ok = all(torch.equal(h["out"].view(torch.int32), L["out"].cpu().view(torch.int32))
                     for L, h in zip(layers, host))
    else:
        e2e_ok = max(pkg.normalized_max_diff(h["out"].numpy(), L["out"].cpu().numpy())
                     for L, h in zip(layers, host))
    pcie = pcie_probe(dev, stream)
    e2e = {"value": flops_step * world / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOPS",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}
    detail["e2e"] = dict(e2e, ms_per_step=e2e_ms, pcie_gbs=pcie,
                         copy_bound_ms_per_step=max(h2d, d2h) / (pcie["bidir_each_gbs"] * 1e9) * 1e3,
                         path="paper_2306_14316_b200.conv_im2win_opt_host_batch -> im2win_conv_host_submit (C ABI), "
                              "pinned host operands, chunked upload/compute/download overlap across layers",
                         equal_to_device_path=e2e_ok,
                         host_buffers="pinned" if all(h["x"].is_pinned() for h in host) else "pageable")
    del host

    # ---- tensor-core peaks (roofline denominators) ----
    tp = tensor_peaks(dev, stream)
    tpk = {"bf16": peaks.get("bf16_tflops") or tp["bf16"], "tf32": tp["tf32"]}
    detail["peaks"].update({"bf16_cublas_tflops_this_run": tp["bf16"], "tf32_cublas_tflops_this_run": tp["tf32"],
                            "tensor_peak_used": tpk,
                            "tensor_peak_note": "bf16: MEASURED_PEAKS.json burst; tf32: cuBLAS 8192^3 in this run"})
    if tc_step:
        for name, rec in per_layer.items():
            cfg = next(L["cfg"] for L in layers if L["name"] == name)
            rec["roofline"] = roofline_row(cfg.flops, tc_min_bytes(cfg, args.variant),
                                           (rec["transform_ms"] + rec["conv_ms"]) * 1e-3, tpk[args.variant],
                                           peaks["hbm_gbs"])

    # ---- tensor-core legs of BASELINE configs 4 and 5 (all ranks; max over ranks) ----
    if not args.no_tc:
        tc = {"tolerance": {"tf32": "max|d|/rms(ref) <= 1e-2", "bf16": "max|d|/rms(ref) <= 4e-2"},
              "note": "production path (direct kernel, or the one-call im2win_conv_fused_nchw: channels-last copy "
                      "inside the conv kernel or by the copy kernel first, then the fused/shift/phase kernel); "
                      "s = the whole call, conv_s = the conv kernel alone on an existing copy; max over ranks; "
                      "roofline = min(tensor peak, AI x HBM) with AI on the minimal bytes (NCHW f32 in + filter + "
                      "NCHW f32 out)"}
        for v in ("tf32", "bf16"):
            traffic = load_tc_traffic(v)
            tc[v] = {}
            for leg, global_n, leg_names in (("config4_n1024", 1024, ("conv9", "conv10", "conv11", "conv12")),
                                             ("config5_n2048", 2048, tuple(names))):
                rows = {}
                tot_f = tot_s = 0.0
                for name in leg_names:
                    cfg = replace(BENCHMARKS[name], batch=global_n, seed=4000 + list(BENCHMARKS).index(name))
                    r = tc_layer(D, cfg, v)
                    row = {"tflops": cfg.flops / r["s"] / 1e12, "tflops_conv_only": cfg.flops / r["conv_s"] / 1e12,
                           "ms": r["s"] * 1e3, "conv_ms": r["conv_s"] * 1e3, "path": r["path"],
                           "per_rank_batch": r["per_rank_batch"], "peak_mem_bytes_rank": r["peak_mem_bytes_rank"]}
                    row["roofline"] = roofline_row(cfg.flops, tc_min_bytes(cfg, v), r["s"], tpk[v], peaks["hbm_gbs"])
                    row["roofline"]["peak_tflops"] = tpk[v]
                    if traffic and name in traffic["layers"]:
                        # ncu bytes at N=128 per GPU, scaled to this call's per-rank batch
                        t = traffic["layers"][name]
                        row["roofline"]["traffic_bytes_rank"] = t["dram_bytes"] * r["per_rank_batch"] / 128
                        row["roofline"]["traffic_source"] = traffic["source"]
                    else:
                        row["roofline"]["traffic_bytes_rank"] = None
                    rows[name] = row
                    tot_f += cfg.flops
                    tot_s += r["s"]
                tc[v][leg] = {"layers": rows, "tflops": tot_f / tot_s / 1e12}
        detail["tensor_core"] = tc

    # ---- rank 0 extras: FMA variant, configs 1/3, cuDNN / im2col+cuBLAS, footprints, CPU oracle ----
    cpu_baseline = None
    if rank == 0 and not args.no_baselines:
        detail["baselines"] = baselines(args, dev, stream, layers, per_layer, pkg, set_fp32_precision)
        detail["other_configs"] = other_configs(args, dev, stream, pkg, peaks)
        if world == 1:
            cpu_baseline = cpu_oracle(layers)
            detail["cpu_baseline"] = cpu_baseline

    # ---- the compact driver line ----
    fp32_nchw = not tc_step and not any("mid" in L for L in layers)
    traffic = load_traffic(names, args.batch, args.variant, "nchw" if fp32_nchw else "windows") if not tc_step else None
    if tc_step:
        pk = tpk[args.variant]
        roof = {"bound": "tensor", "kernel": "tcgen05 conv (per-layer kernels in detail)",
                "achieved": flops_step / (conv_ms_total * 1e-3) / 1e12, "peak": pk, "unit": "TFLOP/s",
                "traffic": None}
    else:
        pk = fp["exact"] if args.variant == "fp32-exact" else fp["ffma"]
        roof = {"bound": "fp32-simt", "kernel": "conv_simt_kernel " + ("exact mul-then-add, packed FFMA2 pairs"
                                                                        if args.variant == "fp32-exact" else "FFMA")
                + (", windows gathered from NCHW" if fp32_nchw else ""),
                "achieved": flops_step / (conv_ms_total * 1e-3) / 1e12, "peak": pk, "unit": "TFLOP/s",
                "traffic": traffic and traffic["conv_bytes_per_launch"]}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["conv_share"] = conv_ms_total / (conv_ms_total + tr_ms_total)
    detail["roofline"] = dict(roof, traffic_detail=traffic,
                              peak_source="FP32: im2win_bench_fp32_peak in this run (148x8 CTAs of independent "
                                          "chains; exact = max of scalar FMUL+FADD and the packed FFMA2 pair form)",
                              achieved_note="sum of the step's conv FLOPs / sum of the conv calls' mean durations "
                                            "(CUDA events inside the timed region)")
    cpu_short = None
    if cpu_baseline is not None:
        cpu_short = {k: cpu_baseline[k] for k in ("value", "unit", "cores", "kind")}
        cpu_short["sample"] = "12 layers at N=1 (per-image slice), oracle port, all host threads"
    tc_summary = None
    if "tensor_core" in detail:
        tc_summary = {f"{v}_{leg[:7]}": round(detail["tensor_core"][v][leg]["tflops"], 1)
                      for v in ("tf32", "bf16") for leg in ("config4_n1024", "config5_n2048")}
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": {"fp32-exact": "f32", "fp32-fma": "f32", "tf32": "tf32", "bf16": "bf16"}[
            args.variant], "data": "synthetic N(0,1), torch.randn on device (seeded)",
        "config": {"workload": (f"paper 12 conv layers, conv_im2win_opt {args.variant} (im2win windows gathered from "
                                f"NCHW, no Ĩ pass), N={args.batch}/GPU" if fp32_nchw else
                                f"paper 12 conv layers, im2win transform + {args.variant} conv, N={args.batch}/GPU"),
                   "global_batch": args.batch * world, "parallelism": f"batch-shard x{world}, no data-path collective",
                   "l2": "no flush: ~15 GB working set per step >> 126 MB L2"},
        "roofline": {k: (round(v, 4) if isinstance(v, float) else v) for k, v in roof.items()},
        "cpu_baseline": cpu_short,
        "e2e": e2e,
        "gpu_launches": gpu_launches,
        "clocks": {k: clocks.get(k) for k in ("sm_mhz", "sm_max_mhz", "reasons")},
        "devices_distinct": D.devices_distinct,
        "tc_tflops": tc_summary,
        "detail": args.detail,
    }
    if rank == 0:
        p = Path(args.detail)
        if not p.is_absolute():
            p = ROOT / p
        p.parent.mkdir(parents=True, exist_ok=True)
        p.write_text(json.dumps(dict(detail, line=line), indent=1) + "\n")
    D.close()
    if rank == 0:
        s = json.dumps(line)
        if len(s) > LINE_LIMIT:  # never let the driver's stdout tail cut the line
            line.pop("tc_tflops")
            s = json.dumps(line)
        print(s, flush=True)


def baselines(args, dev, stream, layers, per_layer, pkg, set_prec) -> dict:
    """cuDNN (FP32 ieee / TF32 / BF16) and im2col+cuBLAS on the same B200, with peak memory."""
    import torch
    import torch.nn.functional as F

    torch.backends.cudnn.benchmark = True
    out = {}

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize(dev)
        best = 1e30
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize(dev)
            best = min(best, a.elapsed_time(b))
        return best

    def peak_mem(fn):
        torch.cuda.synchronize(dev)
        base = torch.cuda.memory_allocated(dev)
        torch.cuda.reset_peak_memory_stats(dev)
        r = fn()
        torch.cuda.synchronize(dev)
        del r
        return torch.cuda.max_memory_allocated(dev) - base

    for L in layers:
        cfg = L["cfg"]
        rec = {}
        cudnn = lambda: F.conv2d(L["x"], L["f"], stride=cfg.stride)  # noqa: E731

        def im2col_cublas():
            cols = F.unfold(L["x"], (cfg.h_f, cfg.w_f), stride=cfg.stride)  # (N, K, L) full batch
            return torch.matmul(L["f"].view(cfg.c_out, -1), cols)

        def im2col_per_image():
            # the reference's im2col route lowers one image at a time (kernels/reference.py:127-137)
            o = torch.empty_like(L["out"])
            fm = L["f"].view(cfg.c_out, -1)
            for i in range(min(cfg.batch, 2)):
                cols = F.unfold(L["x"][i:i + 1], (cfg.h_f, cfg.w_f), stride=cfg.stride)[0]
                torch.matmul(fm, cols, out=o[i].view(cfg.c_out, -1))
            return o

        set_prec("ieee")
        t_cudnn = timed(cudnn)
        rec["cudnn_fp32_tflops"] = cfg.flops / (t_cudnn * 1e-3) / 1e12
        rec["im2col_cublas_tflops"] = cfg.flops / (timed(im2col_cublas) * 1e-3) / 1e12
        if args.variant == "fp32-exact":
            rec["cudnn_fp32_max_rel_diff"] = max_rel_diff_device(cudnn(), L["out"])
        set_prec("tf32")
        rec["cudnn_tf32_tflops"] = cfg.flops / (timed(cudnn) * 1e-3) / 1e12
        set_prec("ieee")
        xb, fb = L["x"].to(torch.bfloat16), L["f"].to(torch.bfloat16)
        rec["cudnn_bf16_tflops"] = cfg.flops / (timed(lambda: F.conv2d(xb, fb, stride=cfg.stride)) * 1e-3) / 1e12
        del xb, fb
        ours = {v: (lambda v=v: pkg.conv_im2win_opt(L["x"], L["f"], cfg.params, variant=v))
                for v in ("fp32-exact", "bf16")}
        # bytes the call allocates beyond its operands (input, filter): output + layout data + workspace
        rec["peak_mem_bytes"] = {"im2win_fp32": peak_mem(ours["fp32-exact"]), "im2win_bf16": peak_mem(ours["bf16"]),
                                 "cudnn_fp32": peak_mem(cudnn), "im2col_cublas_full_batch": peak_mem(im2col_cublas),
                                 "im2col_cublas_per_image": peak_mem(im2col_per_image)}
        rec["footprint_elems"] = {"raw": cfg.elems("raw"), "im2col": cfg.elems("im2col"),
                                  "im2win": cfg.elems("im2win")}
        torch.cuda.empty_cache()
        out[L["name"]] = rec
    tot = sum(L["cfg"].flops for L in layers)

    def step_tf(key):
        return tot / sum(L["cfg"].flops / (out[L["name"]][key] * 1e12) for L in layers) / 1e12

    out["step_tflops"] = {k: step_tf(k) for k in ("cudnn_fp32_tflops", "im2col_cublas_tflops", "cudnn_tf32_tflops",
                                                   "cudnn_bf16_tflops")}
    out["note"] = ("torch FP32 with fp32_precision='ieee' (cuDNN picks its fastest algorithm incl. Winograd/FFT, "
                   "benchmark=True); tf32: fp32_precision='tf32'; bf16: bf16 operands.  peak_mem: bytes allocated by "
                   "the call beyond its operands (the per-image im2col column buffer is reused across images)")
    return out


def other_configs(args, dev, stream, pkg, peaks) -> dict:
    """BASELINE configs 1 (pad 1, native padding) and 3 (conv1 at N=256) on this GPU, headline variant."""
    import torch

    from paper_2306_14316_b200.workloads import BENCHMARKS

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize(dev)
        best = 1e30
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize(dev)
            best = min(best, a.elapsed_time(b))
        return best

    out = {}
    g1 = torch.Generator(device=dev).manual_seed(0)
    p1 = pkg.ConvParams(64, 64, 3, 3, 1, pad=1)
    x1 = torch.randn((8, 64, 56, 56), device=dev, generator=g1)
    f1 = torch.randn((64, 64, 3, 3), device=dev, generator=g1)
    fl1 = 2 * 8 * 64 * 56 * 56 * 64 * 9
    for v in (args.variant, "bf16"):
        t = timed(lambda: pkg.conv_im2win_opt(x1, f1, p1, variant=v))
        out[f"config1_n8_pad1_{v}"] = {"tflops": fl1 / (t * 1e-3) / 1e12, "ms": t}
    c3 = replace(BENCHMARKS["conv1"], batch=256, seed=3)
    g3 = torch.Generator(device=dev).manual_seed(3)
    x3 = torch.randn((256, 3, 227, 227), device=dev, generator=g3)
    f3 = torch.randn((96, 3, 11, 11), device=dev, generator=g3)
    h3, _ = c3.out_dims
    wn3 = torch.empty((256, 3, h3, 11 * c3.w_eff), device=dev)
    from paper_2306_14316_b200.layouts import im2win_into

    t_tr = timed(lambda: im2win_into(x3, wn3, c3.params))
    out["config3_conv1_n256_transform"] = {"ms": t_tr, "gbs": c3.transform_bytes() / (t_tr * 1e-3) / 1e9,
                                           "frac_of_hbm": c3.transform_bytes() / (t_tr * 1e-3) / 1e9
                                           / peaks["hbm_gbs"]}
    for v in (args.variant, "tf32", "bf16"):
        t = timed(lambda: pkg.conv_im2win_opt(x3, f3, c3.params, variant=v))
        out[f"config3_conv1_n256_{v}"] = {"tflops": c3.flops / (t * 1e-3) / 1e12, "ms": t}
    del x1, f1, x3, f3, wn3
    torch.cuda.empty_cache()
    return out


def cpu_oracle(layers) -> dict:
    """The oracle port on the host cores, bounded sample (12 layers at N=1 image, ~10 s)."""
    from oracle import oracle as orc
    from paper_2306_14316_b200.workloads import make_inputs

    threads = orc.max_threads()
    cfgs = [replace(L["cfg"], batch=1) for L in layers]
    ops = [make_inputs(c) for c in cfgs]
    t0 = time.perf_counter()
    reps = 0
    while True:
        for c, (inp, flt) in zip(cfgs, ops):
            w = orc.im2win_fill(inp, c.h_f, c.w_f, c.stride, threads)
            orc.conv_from_windows(w, flt, c.stride, c.out_dims[1], threads)
        reps += 1
        if time.perf_counter() - t0 > 10.0 or reps >= 20:
            break
    dt = (time.perf_counter() - t0) / reps
    return {"value": sum(c.flops for c in cfgs) / dt / 1e12, "unit": "TFLOPS", "cores": threads, "kind": "port",
            "sample": f"12 layers at N=1 image, {reps} reps (per-image slice of the workload)"}


if __name__ == "__main__":
    main()
