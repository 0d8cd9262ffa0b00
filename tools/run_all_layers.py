"""Run every benchmark layer's transform + conv once (the bench step, for ncu captures).

    python tools/run_all_layers.py [--batch 128] [--variant fp32-exact] [--warm]
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
ap.add_argument("--batch", type=int, default=128)
ap.add_argument("--variant", default="fp32-exact")
ap.add_argument("--layers", default="all")
args = ap.parse_args()
dev = torch.device("cuda:0")
names = list(BENCHMARKS) if args.layers == "all" else args.layers.split(",")
for name in names:
    cfg = replace(BENCHMARKS[name], batch=args.batch)
    h_out, w_out = cfg.out_dims
    x = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev)
    win = torch.empty((cfg.batch, cfg.c_in, h_out, cfg.h_f * cfg.w_eff), device=dev)
    out = torch.empty((cfg.batch, cfg.c_out, h_out, w_out), device=dev)
    im2win_into(x, win, cfg.params)
    conv_windows_into(win, f, out, cfg.params, cfg.w_eff, None, args.variant)
    torch.cuda.synchronize()
    del x, f, win, out
    torch.cuda.empty_cache()
print("done", ",".join(names))
