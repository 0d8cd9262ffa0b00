"""A/B of the in-kernel channels-last feed against the separate copy kernel.

For each layer and TC variant: time (a) im2win_nchw_to_nhwc + im2win_conv_fused, (b) the conv
alone on an existing copy, (c) im2win_conv_fused_nchw (copy produced inside the conv kernel);
check (c) is bit-identical to (a).

    python tools/feed_ab.py [layers|all] [batch] [variants]
"""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2306_14316_b200 as pkg  # noqa: E402
from paper_2306_14316_b200 import _lib  # noqa: E402
from paper_2306_14316_b200.kernels import (  # noqa: E402
    conv_fused_into,
    conv_fused_nchw_into,
    direct_preferred,
    nhwc_into,
    nhwc_pitch,
)

layers = sys.argv[1].split(",") if len(sys.argv) > 1 and sys.argv[1] != "all" else list(pkg.BENCHMARKS)
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
variants = sys.argv[3].split(",") if len(sys.argv) > 3 else ["tf32", "bf16"]
dev = torch.device("cuda:0")


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best


print(f"{'layer':7s} {'var':4s} {'copy+conv ms':>12s} {'conv ms':>8s} {'feed ms':>8s} {'TF copy+conv':>12s} "
      f"{'TF feed':>8s} {'TF conv':>8s} same-bits kernel")
for name in layers:
    cfg = replace(pkg.BENCHMARKS[name], batch=batch)
    h_out, w_out = cfg.out_dims
    for v in variants:
        if direct_preferred((batch, cfg.c_in, cfg.h_in, cfg.w_in), cfg.params, v):
            continue
        g = torch.Generator(device=dev).manual_seed(7)
        x = torch.randn((batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev, generator=g)
        f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev, generator=g)
        dt = torch.bfloat16 if v == "bf16" else torch.float32
        xc = torch.empty((batch, cfg.h_in, cfg.w_in, nhwc_pitch(cfg.c_in, v)), device=dev, dtype=dt)
        o1 = torch.empty((batch, cfg.c_out, h_out, w_out), device=dev)
        o2 = torch.full_like(o1, float("nan"))

        def copy_conv():
            nhwc_into(x, xc)
            conv_fused_into(xc, f, o1, cfg.params, v)

        def conv_only():
            conv_fused_into(xc, f, o1, cfg.params, v)

        def feed():
            conv_fused_nchw_into(x, xc, f, o2, cfg.params, v)

        t_a = timed(copy_conv)
        t_b = timed(conv_only)
        t_c = timed(feed)
        kern = _lib.last_kernel()
        copy_conv()
        feed()
        torch.cuda.synchronize()
        same = bool(torch.equal(o1.view(torch.int32), o2.view(torch.int32)))
        fl = 2.0 * batch * cfg.c_out * h_out * w_out * cfg.c_in * cfg.h_f * cfg.w_f
        print(f"{name:7s} {v:4s} {t_a:12.3f} {t_b:8.3f} {t_c:8.3f} {fl / t_a / 1e9:12.1f} {fl / t_c / 1e9:8.1f} "
              f"{fl / t_b / 1e9:8.1f} {same} {kern}", flush=True)
