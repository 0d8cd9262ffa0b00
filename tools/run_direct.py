"""Run one layer's direct (in-SM im2win) tensor-core conv `reps` times (for ncu captures)."""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_14316_b200.kernels import conv_direct_into  # noqa: E402
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

name, variant = sys.argv[1], sys.argv[2]
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 128
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
cfg = replace(BENCHMARKS[name], batch=batch)
dev = torch.device("cuda:0")
h_out, w_out = cfg.out_dims
x = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev)
o = torch.empty((cfg.batch, cfg.c_out, h_out, w_out), device=dev)
for _ in range(reps):
    conv_direct_into(x, f, o, cfg.params, variant)
torch.cuda.synchronize()
print("done")
