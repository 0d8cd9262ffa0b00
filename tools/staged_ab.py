"""Fused TC kernel epilogue A/B: lane = pixel stores vs the staged aligned-line writer (IM2WIN_STAGED_EPI).

    python tools/staged_ab.py [layers] [batch] [variants]

Times the conv alone (conv_fused_into on an existing channels-last copy), median of 7, both
epilogues in one process (the library reads the switch per launch), and checks the outputs are
bit-identical.
"""
import os
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_14316_b200 import _lib  # noqa: E402
from paper_2306_14316_b200.kernels import conv_fused_into, nhwc_into, nhwc_pitch  # noqa: E402
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

layers = (sys.argv[1] if len(sys.argv) > 1 else "conv3,conv5,conv6,conv7,conv11,conv12").split(",")
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
    ts.sort()
    return ts[len(ts) // 2]


for name in layers:
    cfg = replace(BENCHMARKS[name], batch=batch)
    h_out, w_out = cfg.out_dims
    g = torch.Generator(device=dev).manual_seed(3)
    x = torch.randn((batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev, generator=g)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev, generator=g)
    outs = [torch.empty((batch, cfg.c_out, h_out, w_out), device=dev) for _ in range(2)]
    for v in variants:
        xc = torch.empty((batch, cfg.h_in, cfg.w_in, nhwc_pitch(cfg.c_in, v)), device=dev,
                         dtype=torch.bfloat16 if v == "bf16" else torch.float32)
        nhwc_into(x, xc)
        res = []
        for mode, o in zip(("0", "1"), outs):
            os.environ["IM2WIN_STAGED_EPI"] = mode
            o.fill_(float("nan"))
            t = timed(lambda: conv_fused_into(xc, f, o, cfg.params, v))
            res.append(t)
            kern = _lib.last_kernel()
        os.environ["IM2WIN_STAGED_EPI"] = "0"
        same = bool(torch.equal(outs[0].view(torch.int32), outs[1].view(torch.int32)))
        print(f"{name:6s} {v:5s} N={batch} plain {res[0]:7.3f} ms {cfg.flops / res[0] / 1e9:7.1f} TF | staged "
              f"{res[1]:7.3f} ms {cfg.flops / res[1] / 1e9:7.1f} TF  x{res[0] / res[1]:.3f} same={same} [{kern}]",
              flush=True)
