"""Run one layer's NCHW-direct FP32 conv twice (for per-layer ncu captures): python tools/run_nchw_layer.py conv4 128"""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_14316_b200.kernels import conv_nchw_into  # noqa: E402
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

cfg = replace(BENCHMARKS[sys.argv[1]], batch=int(sys.argv[2]) if len(sys.argv) > 2 else 128)
dev = torch.device("cuda:0")
h_out, w_out = cfg.out_dims
x = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev)
o = torch.empty((cfg.batch, cfg.c_out, h_out, w_out), device=dev)
for _ in range(2):
    conv_nchw_into(x, f, o, cfg.params)
torch.cuda.synchronize()
