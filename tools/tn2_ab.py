"""Phase kernel, one tap per MMA (N=64, 4 tiles/item) vs tap pairs per MMA (N=128, 2 tiles/item):

    python tools/tn2_ab.py [layers] [batch] [variants] [switch] [on-value]

switch: IM2WIN_PHASE_TN2 (default), compared at 0 and the value given last (1 auto, 2 forced).

Conv alone on an existing channels-last copy (median of 7) and the one-call path; error =
max|d| / rms(ref) against the FP32-exact call.  IM2WIN_PHASE_TN2 is read per launch.
"""
import os
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_14316_b200 import _lib  # noqa: E402
from paper_2306_14316_b200.kernels import (conv_fused_into, conv_fused_nchw_into, conv_nchw_into,  # noqa: E402
                                           nhwc_into, nhwc_pitch)
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

layers = (sys.argv[1] if len(sys.argv) > 1 else "conv4,conv9").split(",")
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
variants = (sys.argv[3] if len(sys.argv) > 3 else "bf16,tf32").split(",")
switch = sys.argv[4] if len(sys.argv) > 4 else "IM2WIN_PHASE_TN2"
on = sys.argv[5] if len(sys.argv) > 5 else "1"  # "2": tap pairs wherever legal
dev = torch.device("cuda:0")


def timed(fn, reps=7):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


for name in layers:
    cfg = replace(BENCHMARKS[name], batch=batch)
    h_out, w_out = cfg.out_dims
    g = torch.Generator(device=dev).manual_seed(4)
    x = torch.randn((batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev, generator=g)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev, generator=g)
    ref = torch.empty((batch, cfg.c_out, h_out, w_out), device=dev)
    conv_nchw_into(x, f, ref, cfg.params)
    rms = ref.pow(2).mean().sqrt()
    out = torch.empty_like(ref)
    for v in variants:
        xc = torch.empty((batch, cfg.h_in, cfg.w_in, nhwc_pitch(cfg.c_in, v)), device=dev,
                         dtype=torch.bfloat16 if v == "bf16" else torch.float32)
        nhwc_into(x, xc)
        row = []
        for mode in ("0", on):
            os.environ[switch] = mode
            out.fill_(float("nan"))
            t_conv = timed(lambda: conv_fused_into(xc, f, out, cfg.params, v))
            err = float((out - ref).abs().max() / rms)
            kern = _lib.last_kernel()
            t_one = timed(lambda: conv_fused_nchw_into(x, xc, f, out, cfg.params, v))
            row.append(f"TN2={mode}: conv {t_conv:7.3f} ms {cfg.flops / t_conv / 1e9:6.1f} TF, one-call "
                       f"{cfg.flops / t_one / 1e9:6.1f} TF, err {err:.1e} [{kern[22:]}]")
        os.environ[switch] = "0"
        print(f"{name:6s} {v:5s} N={batch} | " + " | ".join(row), flush=True)
