"""64-byte vs 128-byte K rows in the fused TC kernel (IM2WIN_ROW64 A/B): time and bitwise agreement.

    python tools/row64_ab.py [layers] [batch]
"""
import os
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2306_14316_b200 as pkg  # noqa: E402
from paper_2306_14316_b200 import _lib  # noqa: E402

layers = sys.argv[1].split(",") if len(sys.argv) > 1 else ["conv7"]
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
dev = torch.device("cuda:0")
for name in layers:
    cfg = replace(pkg.BENCHMARKS[name], batch=batch)
    g = torch.Generator(device=dev).manual_seed(5)
    x = torch.randn((batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev, generator=g)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev, generator=g)
    for v in ("tf32", "bf16"):
        res = {}
        for r64 in ("0", "1"):
            os.environ["IM2WIN_ROW64"] = r64
            o = pkg.conv_im2win_opt(x, f, cfg.params, variant=v, tc_path="fused").data.clone()
            k = _lib.last_kernel()
            torch.cuda.synchronize()
            ts = []
            for _ in range(9):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                pkg.conv_im2win_opt(x, f, cfg.params, variant=v, tc_path="fused")
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ts.sort()
            res[r64] = (o, ts[4], k)
        same = torch.equal(res["0"][0].view(torch.int32), res["1"][0].view(torch.int32))
        close = torch.allclose(res["0"][0], res["1"][0], rtol=0, atol=0)
        fl = cfg.flops
        print(f"{name} N={batch} {v}: 128B rows {res['0'][1]:.3f} ms ({fl / res['0'][1] / 1e9:.1f} TF), "
              f"64B rows {res['1'][1]:.3f} ms ({fl / res['1'][1] / 1e9:.1f} TF), bitwise={same} equal={close}; "
              f"{res['1'][2]}", flush=True)
