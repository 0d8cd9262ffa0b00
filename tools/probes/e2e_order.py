"""e2e step time of the streamed host path: original layer order vs the batch API's order."""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import torch  # noqa: E402

import paper_2306_14316_b200 as pkg  # noqa: E402
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

layers = []
for name, c in BENCHMARKS.items():
    cfg = replace(c, batch=128)
    h_out, w_out = cfg.out_dims
    layers.append((cfg, torch.randn((128, cfg.c_in, cfg.h_in, cfg.w_in)).pin_memory(),
                   torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f)).pin_memory(),
                   torch.empty((128, cfg.c_out, h_out, w_out)).pin_memory()))
flops = sum(c.flops for c, *_ in layers)


def in_order():
    hs = [pkg.conv_im2win_opt_host(x, f, c.params, out=o, wait=False) for c, x, f, o in layers]
    for h in hs:
        h.wait()


def batch():
    pkg.conv_im2win_opt_host_batch([(x, f, c.params) for c, x, f, o in layers], outs=[o for *_, o in layers])


for name, fn in (("in_order", in_order), ("batch", batch), ("in_order", in_order)):
    fn()
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name:9s} {best:7.1f} ms/step  {flops / best / 1e9:6.2f} TFLOPS", flush=True)
