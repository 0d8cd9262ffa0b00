"""FP32-exact NCHW-direct conv per compiled CTA tile (explicit TilePlans) next to the library's own
choice: python tools/nchw_tile_sweep.py [layers] [batch]"""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2306_14316_b200 as pkg  # noqa: E402
from paper_2306_14316_b200 import _lib  # noqa: E402
from paper_2306_14316_b200.kernels import conv_nchw_into  # noqa: E402

layers = (sys.argv[1] if len(sys.argv) > 1 else "conv12,conv1,conv2,conv3,conv6,conv10").split(",")
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
dev = torch.device("cuda:0")
plans = [("auto", None)] + [(f"{bm}x{bn} 8x8", pkg.TilePlan(bm, bn, 8, 8, 8)) for bm, bn in pkg.plan.SIMT_TILES] + \
        [(f"{bm}x{bn} 4x4", pkg.TilePlan(bm, bn, 8, 4, 4)) for bm, bn in pkg.plan.SIMT_TILES_MT4]
for name in layers:
    cfg = replace(pkg.BENCHMARKS[name], batch=batch)
    h_out, w_out = cfg.out_dims
    x = torch.randn((batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev)
    o = torch.empty((batch, cfg.c_out, h_out, w_out), device=dev)
    row = []
    for label, plan in plans:
        conv_nchw_into(x, f, o, cfg.params, plan)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            conv_nchw_into(x, f, o, cfg.params, plan)
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / 5
        row.append(f"{label} {cfg.flops / t / 1e9:5.1f}")
        if plan is None:
            row[-1] += f" [{_lib.last_kernel()}]"
    print(f"{name:6s} " + " | ".join(row), flush=True)
