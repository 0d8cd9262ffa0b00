"""Few-channel TC layers: channels-last copy + conv vs the row-stacked copy + 1 x Wf conv (IM2WIN_STACK):

    python tools/stack_ab.py [layers] [batch] [variants]

ms per one-call conv (median of 7), error = max|d| / rms(ref) against the FP32-exact call.
"""
import os
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_14316_b200 import _lib  # noqa: E402
from paper_2306_14316_b200.kernels import conv_fused_nchw_into, conv_nchw_into, nhwc_pitch  # noqa: E402
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

layers = (sys.argv[1] if len(sys.argv) > 1 else "conv3,conv7").split(",")
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
variants = (sys.argv[3] if len(sys.argv) > 3 else "bf16,tf32").split(",")
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
    g = torch.Generator(device=dev).manual_seed(8)
    x = torch.randn((batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev, generator=g)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev, generator=g)
    ref = torch.empty((batch, cfg.c_out, h_out, w_out), device=dev)
    conv_nchw_into(x, f, ref, cfg.params)
    rms = ref.pow(2).mean().sqrt()
    out = torch.empty_like(ref)
    for v in variants:
        esz = 2 if v == "bf16" else 4
        nb = max(batch * cfg.h_in * cfg.w_in * nhwc_pitch(cfg.c_in, v),
                 batch * h_out * cfg.w_in * nhwc_pitch(cfg.c_in * cfg.h_f, v)) * esz
        scratch = torch.empty(nb, dtype=torch.uint8, device=dev)
        row = []
        for mode in ("0", "2"):
            os.environ["IM2WIN_STACK"] = mode
            out.fill_(float("nan"))
            t = timed(lambda: conv_fused_nchw_into(x, scratch, f, out, cfg.params, v))
            err = float((out - ref).abs().max() / rms)
            row.append(f"{'copy' if mode == '0' else 'stacked'} {t:7.3f} ms {cfg.flops / t / 1e9:6.1f} TF err {err:.1e} "
                       f"[{_lib.last_kernel()[21:60]}]")
        os.environ["IM2WIN_STACK"] = "0"
        print(f"{name:6s} {v:5s} N={batch} | " + " | ".join(row), flush=True)
