"""Sweep chunk size for the streamed host path over the 12-layer step (N=128).

    IM2WIN_HOST_DEPTH=3 python tools/e2e_sweep.py 8,16,32
"""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2306_14316_b200 as pkg  # noqa: E402
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

chunks = [int(c) for c in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0]
dev = torch.device("cuda:0")
layers = []
for name, c in BENCHMARKS.items():
    cfg = replace(c, batch=128)
    h_out, w_out = cfg.out_dims
    layers.append((cfg, torch.randn((128, cfg.c_in, cfg.h_in, cfg.w_in)).pin_memory(),
                   torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f)).pin_memory(),
                   torch.empty((128, cfg.c_out, h_out, w_out)).pin_memory()))
flops = sum(c.flops for c, *_ in layers)
for ch in chunks:
    def step():
        jobs = [pkg.conv_im2win_opt_host(x, f, c.params, out=o, chunk_images=ch, wait=False) for c, x, f, o in layers]
        for j in jobs:
            j.wait()
    step()
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"chunk={ch:3d} {best:7.1f} ms/step  {flops / best / 1e9:6.2f} TFLOPS", flush=True)
