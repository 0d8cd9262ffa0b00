"""One fused-NCHW (in-kernel feed) conv call for ncu: python tools/run_feed.py layer batch variant [feed]"""
import os
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2306_14316_b200 as pkg  # noqa: E402
from paper_2306_14316_b200.kernels import conv_fused_into, conv_fused_nchw_into, nhwc_into, nhwc_pitch  # noqa: E402

name, batch, v = sys.argv[1], int(sys.argv[2]), sys.argv[3]
feed = len(sys.argv) <= 4 or sys.argv[4] != "0"
cfg = replace(pkg.BENCHMARKS[name], batch=batch)
dev = torch.device("cuda:0")
h_out, w_out = cfg.out_dims
x = torch.randn((batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev)
xc = torch.empty((batch, cfg.h_in, cfg.w_in, nhwc_pitch(cfg.c_in, v)), device=dev,
                 dtype=torch.bfloat16 if v == "bf16" else torch.float32)
o = torch.empty((batch, cfg.c_out, h_out, w_out), device=dev)
for _ in range(2):
    if feed:
        conv_fused_nchw_into(x, xc, f, o, cfg.params, v)
    else:
        nhwc_into(x, xc)
        conv_fused_into(xc, f, o, cfg.params, v)
torch.cuda.synchronize()
