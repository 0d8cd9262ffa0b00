"""Copy rate of the feed warps' code alone vs the copy kernel: python tools/feed_probe.py layer batch"""
import os
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2306_14316_b200 as pkg  # noqa: E402
from paper_2306_14316_b200.kernels import nhwc_into, nhwc_pitch  # noqa: E402

dev = torch.device("cuda:0")
for name in sys.argv[1].split(","):
    batch = int(sys.argv[2])
    cfg = replace(pkg.BENCHMARKS[name], batch=batch)
    x = torch.randn((batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
    for v in ("bf16", "tf32"):
        xc = torch.empty((batch, cfg.h_in, cfg.w_in, nhwc_pitch(cfg.c_in, v)), device=dev,
                         dtype=torch.bfloat16 if v == "bf16" else torch.float32)
        nbytes = x.numel() * 4 + xc.numel() * xc.element_size()
        row = [f"{name} {v}"]
        ref = None
        for probe in ("0", "148", "296", "592"):
            os.environ["IM2WIN_FEED_PROBE"] = probe
            nhwc_into(x, xc)
            torch.cuda.synchronize()
            if ref is None:
                ref = xc.clone()
            same = torch.equal(ref.view(torch.int16) if v == "bf16" else ref.view(torch.int32),
                               xc.view(torch.int16) if v == "bf16" else xc.view(torch.int32))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                nhwc_into(x, xc)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 10
            row.append(f"grid {probe}: {ms:.3f} ms {nbytes / ms / 1e6:.0f} GB/s {'ok' if same else 'DIFF'}")
        print(" | ".join(row), flush=True)
os.environ["IM2WIN_FEED_PROBE"] = "0"
