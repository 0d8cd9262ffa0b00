"""Channels-last copy time per kernel choice: python tools/copy_ab.py [layers] [batch]
(IM2WIN_COPY_BLOCK=0 forces the 32x32 generic kernel where the small-image block kernel applies)."""
import os
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_14316_b200.kernels import nhwc_into, nhwc_pitch  # noqa: E402
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

layers = (sys.argv[1] if len(sys.argv) > 1 else "conv12").split(",")
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
dev = torch.device("cuda:0")
for name in layers:
    cfg = replace(BENCHMARKS[name], batch=batch)
    x = torch.randn((batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
    for v in ("bf16", "tf32"):
        xc = torch.empty((batch, cfg.h_in, cfg.w_in, nhwc_pitch(cfg.c_in, v)), device=dev,
                         dtype=torch.bfloat16 if v == "bf16" else torch.float32)
        nbytes = x.numel() * 4 + xc.numel() * xc.element_size()
        row = []
        for mode in ("0", "1"):
            os.environ["IM2WIN_COPY_BLOCK"] = mode
            nhwc_into(x, xc)
            torch.cuda.synchronize()
            ts = []
            for _ in range(9):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                nhwc_into(x, xc)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            t = sorted(ts)[4]
            row.append(f"{'generic' if mode == '0' else 'block'} {t * 1e3:7.1f} us {nbytes / t / 1e6:6.0f} GB/s")
        print(f"{name:6s} {v:5s} N={batch} " + " | ".join(row), flush=True)
