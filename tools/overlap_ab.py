"""Chunked copy/conv overlap A/B for the one-call tensor-core path (im2win_conv_fused_nchw):

    python tools/overlap_ab.py [layers] [batch] [variants] [chunks] [sms]
    e.g. python tools/overlap_ab.py conv4,conv8 2048 bf16,tf32 128,256 16,24,32

For each layer/variant: the copy-first call (IM2WIN_OVERLAP=0) and every (chunk, SMs) setting, ms
(median of 5 after a warm-up), TFLOPS, and whether the output is bit-identical to the copy-first
call.  The library reads the switches per call, so one process runs every setting.
"""
import os
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_14316_b200 import _lib  # noqa: E402
from paper_2306_14316_b200.kernels import conv_fused_nchw_into  # noqa: E402
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

layers = (sys.argv[1] if len(sys.argv) > 1 else "conv4").split(",")
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
variants = (sys.argv[3] if len(sys.argv) > 3 else "bf16").split(",")
chunks = [int(c) for c in (sys.argv[4] if len(sys.argv) > 4 else "256").split(",")]
sms = [int(c) for c in (sys.argv[5] if len(sys.argv) > 5 else "24").split(",")]
dev = torch.device("cuda:0")


def timed(fn, reps=5):
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
    g = torch.Generator(device=dev).manual_seed(5)
    x = torch.randn((batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev, generator=g)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev, generator=g)
    ref = torch.empty((batch, cfg.c_out, h_out, w_out), device=dev)
    out = torch.empty_like(ref)
    for v in variants:
        bf = v == "bf16"
        pitch = -(-cfg.c_in // (8 if bf else 4)) * (8 if bf else 4)
        xc = torch.empty((batch, cfg.h_in, cfg.w_in, pitch), device=dev, dtype=torch.bfloat16 if bf else torch.float32)
        os.environ["IM2WIN_OVERLAP"] = "0"
        t0 = timed(lambda: conv_fused_nchw_into(x, xc, f, ref, cfg.params, v))
        print(f"{name:6s} {v:5s} N={batch} copy-first      {t0:8.3f} ms {cfg.flops / t0 / 1e9:7.1f} TF  "
              f"{_lib.last_kernel()}", flush=True)
        for ch in chunks:
            for k in sms:
                os.environ["IM2WIN_OVERLAP"] = str(ch)
                os.environ["IM2WIN_OVERLAP_SMS"] = str(k)
                out.fill_(float("nan"))
                t = timed(lambda: conv_fused_nchw_into(x, xc, f, out, cfg.params, v))
                same = bool(torch.equal(out.view(torch.int32), ref.view(torch.int32)))
                print(f"{name:6s} {v:5s} N={batch} chunk {ch:4d} sms {k:3d} {t:8.3f} ms {cfg.flops / t / 1e9:7.1f} TF  "
                      f"same={same}  x{t0 / t:.3f}", flush=True)
        os.environ["IM2WIN_OVERLAP"] = "0"
        del xc
    del x, f, ref, out
    torch.cuda.empty_cache()
