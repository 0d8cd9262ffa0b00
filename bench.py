#!/usr/bin/env python
"""Benchmark: im2win transform + convolution over the paper's 12 layers on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A *step* is one pass of the hot path (im2win transform + FP32-exact im2win
convolution) over all twelve benchmark layers (BASELINE.json configs[1]:
/root/reference/pkg/src/winconv/bench.py:88-104) at N=128 images per GPU.
`value` = total algorithmic FLOPs of all ranks / max-over-ranks device time
(TFLOPS, FLOPs = 2*N*Co*Ho*Wo*Ci*Hf*Wf as in winconv bench.py:70-74; the
transform is inside the timed region, as in the reference's TFLOPS, bench.py:259).
Multi-GPU is batch sharding (weak scaling: each rank owns its own 128-image
slice), no collective on the data path.

`--impl reference` times the CPU oracle (a C restatement of the reference's
algorithm, oracle/) on a bounded sample of the same workload on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from dataclasses import replace
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}


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


def load_traffic(names, batch: int, variant: str):
    """DRAM traffic of the step's kernels from the committed ncu --set full capture.

    profiles/r01_traffic_n128.json is written by tools/ncu_traffic.py from one
    `ncu --set full` capture per layer (dram__bytes_read.sum + dram__bytes_write.sum).
    Returns None when it does not cover this workload.
    """
    p = ROOT / "profiles" / "r01_traffic_n128.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    if d.get("batch") != batch or d.get("variant") != variant or not all(n in d["layers"] for n in names):
        return None
    conv = [d["layers"][n]["conv_dram_bytes"] for n in names]
    xf = [d["layers"][n]["transform_dram_bytes"] for n in names]
    alg = [d["layers"][n]["conv_algorithmic_bytes"] for n in names]
    return {"source": str(p.relative_to(ROOT)), "capture": d.get("capture"),
            "conv_bytes_per_launch": sum(conv) / len(conv),
            "per_launch_note": "per layer conv call (mean over the 12 layers); a tail-split layer's two "
                               "kernel launches count as one call",
            "conv_algorithmic_bytes_per_launch": sum(alg) / len(alg),
            "transform_bytes_per_launch": sum(xf) / len(xf),
            "per_layer": {n: d["layers"][n] for n in names}}


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
    sample = (f"12 paper layers at N={sample_batch} image per step (the N=128 workload's per-image slice; "
              f"images are independent), im2win transform + unfused-f32 window conv")
    line = {
        "metric": "TFLOPS per conv layer (12 benchmarks) at 1/2/4/8 B200; memory footprint",
        "impl": "reference", "value": value, "unit": "TFLOPS", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic N(0,1), numpy PCG64 seeded",
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


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=128, help="images per GPU")
    ap.add_argument("--variant", default="fp32-exact")
    ap.add_argument("--layers", default="all")
    ap.add_argument("--no-baselines", action="store_true", help="skip cuDNN / im2col+cuBLAS / CPU legs")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-tc", action="store_true", help="skip the TF32/BF16 tensor-core section")
    args = ap.parse_args()

    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2306_14316_b200 as pkg
    from paper_2306_14316_b200 import _lib
    from paper_2306_14316_b200.kernels import conv_windows_into
    from paper_2306_14316_b200.layouts import im2win_into
    from paper_2306_14316_b200.workloads import BENCHMARKS

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU over NCCL; IM2WIN_DIST_BACKEND=gloo lets several ranks share one GPU
    # (exercises the multi-rank path -- barrier, max over ranks, rank-0 line -- on a 1-GPU box)
    backend = os.environ.get("IM2WIN_DIST_BACKEND", "nccl")
    dev = torch.device("cuda", local_rank % torch.cuda.device_count() if world > 1 else 0)
    if world > 1:
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(dev)
    set_fp32_precision("ieee")

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    names = list(BENCHMARKS) if args.layers == "all" else args.layers.split(",")
    peaks = load_peaks()

    # ---- allocate per-layer operands once (inputs resident in HBM) ----
    gen = torch.Generator(device=dev)
    layers = []
    for i, name in enumerate(names):
        cfg = replace(BENCHMARKS[name], batch=args.batch, seed=1000 + i + 97 * rank)
        gen.manual_seed(cfg.seed)
        h_out, w_out = cfg.out_dims
        x = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev, generator=gen)
        f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev, generator=gen)
        win = torch.empty((cfg.batch, cfg.c_in, h_out, cfg.h_f * cfg.w_eff), device=dev)
        out = torch.empty((cfg.batch, cfg.c_out, h_out, w_out), device=dev)
        layers.append(dict(name=name, cfg=cfg, x=x, f=f, win=win, out=out))

    def run_layer(L):
        im2win_into(L["x"], L["win"], L["cfg"].params)
        conv_windows_into(L["win"], L["f"], L["out"], L["cfg"].params, L["cfg"].w_eff, None, args.variant)

    def step():
        for L in layers:
            run_layer(L)

    stream = torch.cuda.current_stream(dev)
    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize(dev)

    # ---- timed region: exactly K steps ----
    # Events around every transform and conv launch are recorded inside the timed
    # region (same stream, GPU kept busy by the queue) so the dominant kernel's
    # average launch duration comes from the run that produces `value`.
    n_l = len(layers)
    marks = [[[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n_l)]
             for _ in range(args.steps)]
    sampler = ClockSampler(dev.index)
    sampler.start()
    time.sleep(0.3)
    conv_launches0 = _lib.load().im2win_conv_launch_count()
    barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for k in range(args.steps):
        for L, m in zip(layers, marks[k]):
            m[0].record(stream)
            im2win_into(L["x"], L["win"], L["cfg"].params)
            m[1].record(stream)
            conv_windows_into(L["win"], L["f"], L["out"], L["cfg"].params, L["cfg"].w_eff, None, args.variant)
            m[2].record(stream)
    ev1.record(stream)
    conv_launches = _lib.load().im2win_conv_launch_count() - conv_launches0
    torch.cuda.synchronize(dev)
    barrier()
    clocks = sampler.stop()
    elapsed_ms = max_over_ranks(ev0.elapsed_time(ev1))
    flops_step = sum(L["cfg"].flops for L in layers)
    value = flops_step * world * args.steps / (elapsed_ms * 1e-3) / 1e12
    ms_per_step = elapsed_ms / args.steps

    # ---- per-layer breakdown from the timed region (mean over the K steps) ----
    per_layer = []
    conv_ms_total = 0.0
    tr_ms_total = 0.0
    for li, L in enumerate(layers):
        cfg = L["cfg"]
        t_tr = statistics.fmean(marks[k][li][0].elapsed_time(marks[k][li][1]) for k in range(args.steps))
        t_cv = statistics.fmean(marks[k][li][1].elapsed_time(marks[k][li][2]) for k in range(args.steps))
        conv_ms_total += t_cv
        tr_ms_total += t_tr
        tb = cfg.transform_bytes()
        per_layer.append({
            "name": cfg.name, "batch": cfg.batch, "gflop": cfg.flops / 1e9,
            "transform_ms": t_tr, "conv_ms": t_cv,
            "tflops": cfg.flops / ((t_tr + t_cv) * 1e-3) / 1e12,
            "tflops_conv_only": cfg.flops / (t_cv * 1e-3) / 1e12,
            "transform_gbs": tb / (t_tr * 1e-3) / 1e9,
            "footprint_bytes": {"raw": 4 * cfg.elems("raw"), "im2col": 4 * cfg.elems("im2col"),
                                "im2win": 4 * cfg.elems("im2win")},
        })

    # ---- the FFMA variant (within 1e-4 of the reference, not bit-exact), same step for context ----
    fma = None
    if args.variant == "fp32-exact" and rank == 0:
        fma_out = [torch.empty_like(L["out"]) for L in layers]
        for L, o in zip(layers, fma_out):  # warm-up
            conv_windows_into(L["win"], L["f"], o, L["cfg"].params, L["cfg"].w_eff, None, "fp32-fma")
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(layers) + 1)]
        ev[0].record(stream)
        for i, (L, o) in enumerate(zip(layers, fma_out)):
            im2win_into(L["x"], L["win"], L["cfg"].params)
            conv_windows_into(L["win"], L["f"], o, L["cfg"].params, L["cfg"].w_eff, None, "fp32-fma")
            ev[i + 1].record(stream)
        torch.cuda.synchronize(dev)
        fma = {"step_tflops": flops_step / (ev[0].elapsed_time(ev[-1]) * 1e-3) / 1e12,
               "max_rel_diff_vs_exact": max(max_rel_diff_device(o, L["out"]) for L, o in zip(layers, fma_out)),
               "layers_tflops": {L["cfg"].name: L["cfg"].flops / (ev[i].elapsed_time(ev[i + 1]) * 1e-3) / 1e12
                                 for i, L in enumerate(layers)},
               "note": "transform + FFMA conv (ascending k, one rounding per multiply-add); bounded by the FFMA peak"}
        del fma_out

    # ---- the other BASELINE.json configs on this GPU (rank 0): config 1 (pad 1, native
    # padding) and config 3 (conv1 at N=256, the window-transform stress case) ----
    other_cfgs = None
    if rank == 0:
        from paper_2306_14316_b200.workloads import BENCHMARKS as _B

        def timed_pair(fn_tr, fn_cv, reps=5):
            fn_tr()
            fn_cv()
            torch.cuda.synchronize(dev)
            bt = bc = 1e30
            for _ in range(reps):
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                e[0].record(stream)
                fn_tr()
                e[1].record(stream)
                fn_cv()
                e[2].record(stream)
                torch.cuda.synchronize(dev)
                bt, bc = min(bt, e[0].elapsed_time(e[1])), min(bc, e[1].elapsed_time(e[2]))
            return bt, bc

        other_cfgs = {}
        # config 1: N=8 C=64 56x56 K=64 3x3 s1 pad 1 -> padding inside the transform
        g1 = torch.Generator(device=dev).manual_seed(0)
        p1 = pkg.ConvParams(64, 64, 3, 3, 1, pad=1)
        x1 = torch.randn((8, 64, 56, 56), device=dev, generator=g1)
        f1 = torch.randn((64, 64, 3, 3), device=dev, generator=g1)
        w1 = torch.empty((8, 64, 56, 3 * 58), device=dev)
        o1 = torch.empty((8, 64, 56, 56), device=dev)
        t_tr, t_cv = timed_pair(lambda: im2win_into(x1, w1, p1),
                                lambda: conv_windows_into(w1, f1, o1, p1, 58, None, args.variant))
        fl1 = 2 * 8 * 64 * 56 * 56 * 64 * 9
        other_cfgs["config1_n8_pad1"] = {"tflops": fl1 / ((t_tr + t_cv) * 1e-3) / 1e12,
                                         "tflops_conv_only": fl1 / (t_cv * 1e-3) / 1e12,
                                         "transform_ms": t_tr, "conv_ms": t_cv,
                                         "note": "zero padding inside the transform (ConvParams.pad=1); the "
                                                 "golden checksum of this config is a GPU test"}
        del x1, f1, w1, o1
        # config 3: conv1 (3x227x227, 96x11x11, s4) at N=256
        c3 = replace(_B["conv1"], batch=256, seed=3)
        g3 = torch.Generator(device=dev).manual_seed(3)
        h3, w3o = c3.out_dims
        x3 = torch.randn((256, 3, 227, 227), device=dev, generator=g3)
        f3 = torch.randn((96, 3, 11, 11), device=dev, generator=g3)
        wn3 = torch.empty((256, 3, h3, 11 * c3.w_eff), device=dev)
        o3 = torch.empty((256, 96, h3, w3o), device=dev)
        t_tr, t_cv = timed_pair(lambda: im2win_into(x3, wn3, c3.params),
                                lambda: conv_windows_into(wn3, f3, o3, c3.params, c3.w_eff, None, args.variant))
        other_cfgs["config3_conv1_n256"] = {"tflops": c3.flops / ((t_tr + t_cv) * 1e-3) / 1e12,
                                            "tflops_conv_only": c3.flops / (t_cv * 1e-3) / 1e12,
                                            "transform_ms": t_tr, "conv_ms": t_cv,
                                            "transform_gbs": c3.transform_bytes() / (t_tr * 1e-3) / 1e9,
                                            "transform_frac_of_hbm": c3.transform_bytes() / (t_tr * 1e-3) / 1e9
                                            / peaks["hbm_gbs"]}
        del x3, f3, wn3, o3
        torch.cuda.empty_cache()

    # ---- FP32 CUDA-core peak probe (roofline denominator) ----
    lib = _lib.load()
    sink = torch.empty(256, device=dev)
    peak = {}
    for exact in (1, 0):
        iters, blocks = 1 << 15, 148 * 8
        lib.im2win_bench_fp32_peak(sink.data_ptr(), exact, 256, blocks, stream.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        lib.im2win_bench_fp32_peak(sink.data_ptr(), exact, iters, blocks, stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        peak["exact" if exact else "ffma"] = 2 * 32 * iters * 256 * blocks / (e0.elapsed_time(e1) * 1e-3) / 1e12

    conv_flops = flops_step
    achieved = conv_flops / (conv_ms_total * 1e-3) / 1e12
    traffic = load_traffic(names, args.batch, args.variant)
    pk = peak["exact"] if args.variant == "fp32-exact" else peak["ffma"]
    roofline = {"bound": "fp32-simt", "kernel": "conv_simt_kernel (FMUL+FADD)" if args.variant == "fp32-exact" else args.variant,
                "achieved": achieved, "peak": pk, "unit": "TFLOP/s", "frac": achieved / pk,
                "peak_source": "measured on this box in this run by im2win_bench_fp32_peak "
                               f"({'FMUL+FADD' if args.variant == 'fp32-exact' else 'FFMA'} chains, 148x8 CTAs)",
                "peak_ffma": peak["ffma"], "traffic": traffic and traffic["conv_bytes_per_launch"],
                "traffic_detail": traffic,
                "launches_per_step": {"conv": conv_launches / args.steps, "transform": len(layers),
                                      "pack_filter": len(layers),
                                      "note": "conv > layers: the SIMT tail split runs a layer's last partial wave as a "
                                              "second (4x4-tile) launch; achieved sums both"},
                "achieved_note": "sum of algorithmic FLOPs of the step's conv launches / sum of their mean "
                                 "durations (CUDA events around each launch inside the timed region)",
                "transform": {"bound": "hbm", "achieved": sum(L["cfg"].transform_bytes() for L in layers) / (tr_ms_total * 1e-3) / 1e9,
                              "peak": peaks["hbm_gbs"], "unit": "GB/s", "peak_source": peaks["source"],
                              "traffic": traffic and traffic["transform_bytes_per_launch"],
                              "algorithmic_bytes_per_launch": sum(L["cfg"].transform_bytes() for L in layers) / len(layers)}}
    roofline["transform"]["frac"] = roofline["transform"]["achieved"] / roofline["transform"]["peak"]
    roofline["conv_share_of_step"] = conv_ms_total / (conv_ms_total + tr_ms_total)

    # ---- e2e: public host API (numpy-style call: host operands in, host result out) ----
    # conv_im2win_opt_host streams each layer's batch in chunks (upload / transform+conv /
    # download overlapped on three streams, csrc/pipeline.cu); every byte crosses PCIe inside
    # the timed region.
    e2e = None
    host = []
    for L in layers:
        host.append(dict(x=pinned(L["x"].cpu()), f=pinned(L["f"].cpu()),
                         out=pinned(torch.empty(L["out"].shape, dtype=torch.float32))))
    h2d = sum(h["x"].numel() * 4 + h["f"].numel() * 4 for h in host)
    d2h = sum(h["out"].numel() * 4 for h in host)

    def e2e_step():
        # the 12 layers go through the batch host API: submitted non-blocking (download-heavy
        # layers first, upload-heavy last, so both PCIe directions stay busy), then waited;
        # every output is on the host at the end
        pkg.conv_im2win_opt_host_batch([(h["x"], h["f"], L["cfg"].params) for L, h in zip(layers, host)],
                                       variant=args.variant, outs=[h["out"] for h in host])

    e2e_step()
    torch.cuda.synchronize(dev)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / args.e2e_steps
    # the streamed result must be the device path's result (bitwise), checked once outside the timing
    e2e_ok = all(torch.equal(h["out"].view(torch.int32), L["out"].cpu().view(torch.int32))
                 for L, h in zip(layers, host)) if args.variant == "fp32-exact" else None
    pcie = pcie_probe(dev, stream)
    e2e_bound_ms = max(h2d / (pcie["bidir_each_gbs"] * 1e9), d2h / (pcie["bidir_each_gbs"] * 1e9)) * 1e3
    e2e = {"value": flops_step * world / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOPS",
           "pcie_gbs": pcie, "copy_bound_ms_per_step": e2e_bound_ms,
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
           "path": "paper_2306_14316_b200.conv_im2win_opt_host_batch -> im2win_conv_host_submit (C ABI), pinned "
                   "host operands, chunked upload/compute/download overlap across layers",
           "bitwise_equal_to_device_path": e2e_ok,
           "host_buffers": "pinned" if all(h["x"].is_pinned() and h["out"].is_pinned() for h in host) else "pageable"}
    del host

    # ---- baselines on the same B200 (rank 0): cuDNN and im2col+cuBLAS, FP32 (TF32 off) ----
    baselines = None
    if rank == 0 and not args.no_baselines:
        import torch.nn.functional as F

        torch.backends.cudnn.benchmark = True
        baselines = {}
        for L, rec in zip(layers, per_layer):
            cfg = L["cfg"]

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
                fn()
                torch.cuda.synchronize(dev)
                return torch.cuda.max_memory_allocated(dev) - base

            cudnn = lambda: F.conv2d(L["x"], L["f"], stride=cfg.stride)  # noqa: E731

            def im2col_cublas():
                cols = F.unfold(L["x"], (cfg.h_f, cfg.w_f), stride=cfg.stride)  # (N, K, L)
                return torch.matmul(L["f"].view(cfg.c_out, -1), cols)

            ours = lambda: pkg.conv_im2win_opt(L["x"], L["f"], cfg.params, variant=args.variant)  # noqa: E731
            # true FP32 (IEEE) cuDNN and im2col+cuBLAS, then cuDNN TF32 and BF16 for the TC variants
            set_fp32_precision("ieee")
            t_cudnn = timed(cudnn)
            t_col = timed(im2col_cublas)
            ref = L["out"]  # this layer's fp32-exact output from the timed region (= the reference's bits)
            rec["cudnn_tflops"] = cfg.flops / (t_cudnn * 1e-3) / 1e12
            rec["cudnn_max_rel_diff"] = pkg.max_rel_diff(cudnn(), ref)
            rec["im2col_cublas_tflops"] = cfg.flops / (t_col * 1e-3) / 1e12
            set_fp32_precision("tf32")
            rec["cudnn_tf32_tflops"] = cfg.flops / (timed(cudnn) * 1e-3) / 1e12
            rec["cudnn_tf32_norm_diff"] = pkg.normalized_max_diff(cudnn(), ref)
            set_fp32_precision("ieee")
            xb, fb = L["x"].to(torch.bfloat16), L["f"].to(torch.bfloat16)
            cudnn_bf16 = lambda: F.conv2d(xb, fb, stride=cfg.stride)  # noqa: E731
            rec["cudnn_bf16_tflops"] = cfg.flops / (timed(cudnn_bf16) * 1e-3) / 1e12
            rec["cudnn_bf16_norm_diff"] = pkg.normalized_max_diff(cudnn_bf16().float(), ref)
            del xb, fb
            rec["peak_mem_bytes"] = {"im2win": peak_mem(ours), "cudnn": peak_mem(cudnn),
                                     "im2col_cublas_full_batch": peak_mem(im2col_cublas)}
            torch.cuda.empty_cache()
        tot = sum(L["cfg"].flops for L in layers)

        def step_tf(key):
            return tot / sum(L["cfg"].flops / (r[key] * 1e12) for L, r in zip(layers, per_layer)) / 1e12

        baselines["cudnn_tflops_step"] = step_tf("cudnn_tflops")
        baselines["im2col_cublas_tflops_step"] = step_tf("im2col_cublas_tflops")
        baselines["cudnn_tf32_tflops_step"] = step_tf("cudnn_tf32_tflops")
        baselines["cudnn_bf16_tflops_step"] = step_tf("cudnn_bf16_tflops")
        baselines["note"] = ("cudnn/im2col_cublas: torch FP32 with fp32_precision='ieee' (true FP32; cuDNN picks "
                             "its fastest algorithm, incl. Winograd/FFT, benchmark=True); cudnn_tf32: "
                             "fp32_precision='tf32'; cudnn_bf16: bf16 operands.  *_max_rel_diff / *_norm_diff "
                             "are against the fp32-exact output (the reference's bits)")

    # ---- CPU baseline: the oracle port on the host cores, bounded sample (rank 0, N=1 only) ----
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_baselines:
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
        cpu_baseline = {"value": sum(c.flops for c in cfgs) / dt / 1e12, "unit": "TFLOPS", "cores": threads,
                        "kind": "port", "sample": f"12 layers at N=1 image, {reps} reps (per-image slice of the workload)"}

    # ---- tensor-core variants (rank 0): TF32 / BF16 per layer at N=128 and config 4 ----
    tc = None
    if rank == 0 and not args.no_tc:
        from paper_2306_14316_b200.kernels import (
            conv_direct_into,
            conv_fused_into,
            direct_preferred,
            nhwc_into,
            nhwc_pitch,
        )

        def tc_layer(cfg, v):
            """transform + conv time (ms) of the production TC path for one layer."""
            h_out, w_out = cfg.out_dims
            g2 = torch.Generator(device=dev).manual_seed(cfg.seed)
            x = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev, generator=g2)
            f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev, generator=g2)
            o = torch.empty((cfg.batch, cfg.c_out, h_out, w_out), device=dev)
            # the fused path covers every layer (channel pitch padded to a 16 B multiple)
            w = torch.empty((cfg.batch, cfg.h_in, cfg.w_in, nhwc_pitch(cfg.c_in, v)),
                            dtype=torch.bfloat16 if v == "bf16" else torch.float32, device=dev)
            if direct_preferred(x.shape, cfg.params, v):
                # production choice for this shape: the in-SM im2win kernel reads NCHW directly
                tr = None
                cv = lambda: conv_direct_into(x, f, o, cfg.params, v)  # noqa: E731
                cv()
                path = _lib.last_kernel()
            else:
                tr = lambda: nhwc_into(x, w)  # noqa: E731
                cv = lambda: conv_fused_into(w, f, o, cfg.params, v)  # noqa: E731
                tr()
                cv()
                path = "NHWC copy + " + _lib.last_kernel()
            # each launch sequence is captured in a CUDA graph and replayed 5x between events, so
            # host launch latency (~tens of us per Python call) is not counted as device time
            graphs = []
            for fn in (tr, cv):
                if fn is None:  # no separate transform on this path
                    graphs.append(None)
                    continue
                side = torch.cuda.Stream(dev)
                side.wait_stream(stream)
                with torch.cuda.stream(side):
                    fn()
                stream.wait_stream(side)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, capture_error_mode="relaxed"):
                    fn()
                graphs.append(g)
            torch.cuda.synchronize(dev)
            best = [0.0 if graphs[0] is None else 1e30, 1e30]
            for _ in range(3):
                for i, g in enumerate(graphs):
                    if g is None:
                        continue
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    for _ in range(5):
                        g.replay()
                    b.record(stream)
                    torch.cuda.synchronize(dev)
                    best[i] = min(best[i], a.elapsed_time(b) / 5)
            best_t, best_c = best
            del graphs
            del x, f, o, w
            torch.cuda.empty_cache()
            return best_t, best_c, path

        tc = {"tolerance": {"tf32": "max|d|/rms(ref) <= 1e-2", "bf16": "max|d|/rms(ref) <= 4e-2"},
              "peak_tensor_tflops": {"bf16": peaks.get("bf16_tflops"), "tf32": None,
                                     "source": peaks["source"] + " (tf32: no measured peak; nominal 1100)"}}
        for v in ("tf32", "bf16"):
            rows = {}
            tot_f = tot_ms = 0.0
            for L in layers:
                cfg = L["cfg"]
                t_tr, t_cv, path = tc_layer(cfg, v)
                rows[cfg.name] = {"tflops": cfg.flops / ((t_tr + t_cv) * 1e-3) / 1e12,
                                  "tflops_conv_only": cfg.flops / (t_cv * 1e-3) / 1e12,
                                  "transform_ms": t_tr, "conv_ms": t_cv, "path": path}
                tot_f += cfg.flops
                tot_ms += t_tr + t_cv
            tc[v] = {"layers_n128": rows, "step_tflops_n128": tot_f / (tot_ms * 1e-3) / 1e12}
            # config 4: ResNet-50 3x3 layers (conv9-12) at N=1024 per GPU
            c4 = {}
            for name in ("conv9", "conv10", "conv11", "conv12"):
                cfg = replace(BENCHMARKS[name], batch=1024, seed=4000)
                t_tr, t_cv, path = tc_layer(cfg, v)
                c4[name] = {"tflops": cfg.flops / ((t_tr + t_cv) * 1e-3) / 1e12,
                            "tflops_conv_only": cfg.flops / (t_cv * 1e-3) / 1e12, "path": path}
            tc[v]["config4_n1024"] = c4

    n_layers = len(layers)
    line = {
        "metric": "TFLOPS per conv layer (12 benchmarks) at 1/2/4/8 B200; memory footprint",
        "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic N(0,1) (torch.randn on device, seeded); inputs resident in HBM",
        "config": {"workload": f"paper {n_layers} conv layers (winconv BENCHMARKS), im2win transform + "
                               f"{args.variant} im2win conv per step",
                   "per_gpu_batch": args.batch, "global_batch": args.batch * world,
                   "parallelism": f"batch-shard x{world}, no data-path collective",
                   "variant": args.variant,
                   "l2": "no flush: per-step working set (~15 GB at N=128) >> 126 MB L2"},
        "roofline": roofline,
        "cpu_baseline": cpu_baseline,
        "e2e": e2e,
        # transform + pack_filter per layer per step, plus the conv launches the library counted
        "gpu_launches": 2 * n_layers * args.steps + conv_launches,
        "clocks": clocks,
        "layers": per_layer,
        "baselines": baselines,
        "fp32_fma_variant": fma,
        "other_configs": other_cfgs,
        "tensor_core_variants": tc,
        "peaks": {"fp32_exact_tflops": peak["exact"], "fp32_ffma_tflops": peak["ffma"],
                  "hbm_gbs": peaks["hbm_gbs"], "source": peaks["source"]},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
