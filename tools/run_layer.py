"""Run one benchmark layer's transform + conv a few times (for ncu captures).

    python tools/run_layer.py conv4 --batch 128 --reps 2 [--variant fp32-exact]
"""
import argparse
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2306_14316_b200.kernels import conv_windows_into  # noqa: E402
from paper_2306_14316_b200.layouts import im2win_into  # noqa: E402
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("layer")
ap.add_argument("--batch", type=int, default=128)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--variant", default="fp32-exact")
args = ap.parse_args()
cfg = replace(BENCHMARKS[args.layer], batch=args.batch)
dev = torch.device("cuda:0")
h_out, w_out = cfg.out_dims
x = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev)
win = torch.empty((cfg.batch, cfg.c_in, h_out, cfg.h_f * cfg.w_eff), device=dev)
out = torch.empty((cfg.batch, cfg.c_out, h_out, w_out), device=dev)
for _ in range(args.reps):
    im2win_into(x, win, cfg.params)
    conv_windows_into(win, f, out, cfg.params, cfg.w_eff, None, args.variant)
torch.cuda.synchronize()
print("done", args.layer)
