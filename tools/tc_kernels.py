"""Fused TC conv time per layer under each kernel selection (IM2WIN_PHASE / IM2WIN_SHIFT),
with parity of every selection against the oracle at batch 2.

    python tools/tc_kernels.py [layers|all] [batch]
"""
import os
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2306_14316_b200 as pkg  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2306_14316_b200.kernels import (  # noqa: E402
    conv_direct_into,
    conv_fused_into,
    direct_supported,
    nhwc_into,
    nhwc_pitch,
)

layers = sys.argv[1].split(",") if len(sys.argv) > 1 and sys.argv[1] != "all" else list(pkg.BENCHMARKS)
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
dev = torch.device("cuda:0")
SELECT = {"phase": {"IM2WIN_PHASE": "2", "IM2WIN_SHIFT": "0"}, "shift": {"IM2WIN_PHASE": "0", "IM2WIN_SHIFT": "2"},
          "generic": {"IM2WIN_PHASE": "0", "IM2WIN_SHIFT": "0"}, "auto": {"IM2WIN_PHASE": "1", "IM2WIN_SHIFT": "1"}}


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


for name in layers:
    cfg = pkg.BENCHMARKS[name]
    for v in ("tf32", "bf16"):
        c2 = replace(cfg, batch=2, seed=9)
        inp, flt = pkg.make_inputs(c2)
        ref = orc.conv_direct(inp, flt, c2.stride)
        cb = replace(cfg, batch=batch)
        x = torch.randn((cb.batch, cb.c_in, cb.h_in, cb.w_in), device=dev)
        f = torch.randn((cb.c_out, cb.c_in, cb.h_f, cb.w_f), device=dev)
        h_out, w_out = cb.out_dims
        o = torch.empty((cb.batch, cb.c_out, h_out, w_out), device=dev)
        xc = torch.empty((cb.batch, cb.h_in, cb.w_in, nhwc_pitch(cb.c_in, v)), device=dev,
                         dtype=torch.bfloat16 if v == "bf16" else torch.float32)
        nhwc_into(x, xc)
        row = [f"{name:7s} {v}"]
        for sel, env in SELECT.items():
            os.environ.update(env)
            err = pkg.normalized_max_diff(
                pkg.conv_im2win_opt(inp, flt, c2.params, variant=v, tc_path="fused").numpy(), ref)
            t = timed(lambda: conv_fused_into(xc, f, o, cb.params, v))
            row.append(f"{sel} {cb.flops / t / 1e9:7.1f} TF (err {err:.1e})")
        if direct_supported(x.shape, cb.params, v):
            err = pkg.normalized_max_diff(
                pkg.conv_im2win_opt(inp, flt, c2.params, variant=v, tc_path="direct").numpy(), ref)
            t = timed(lambda: conv_direct_into(x, f, o, cb.params, v))
            row.append(f"direct {cb.flops / t / 1e9:7.1f} TF (err {err:.1e}, no NHWC copy)")
        print("  ".join(row), flush=True)
        del x, f, o, xc
        torch.cuda.empty_cache()
for k in ("IM2WIN_PHASE", "IM2WIN_SHIFT"):
    os.environ.pop(k, None)
