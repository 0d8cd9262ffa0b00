"""conv4 FP32-exact conv time per image across batch sizes around N=128: is the last-wave tail visible?"""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import torch  # noqa: E402

from paper_2306_14316_b200.kernels import conv_windows_into  # noqa: E402
from paper_2306_14316_b200.layouts import im2win_into  # noqa: E402
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "conv4"
for n in [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "120,124,126,127,128,129,130,132").split(",")]:
    cfg = replace(BENCHMARKS[name], batch=n)
    h_out, w_out = cfg.out_dims
    x = torch.randn((n, cfg.c_in, cfg.h_in, cfg.w_in), device="cuda")
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device="cuda")
    win = torch.empty((n, cfg.c_in, h_out, cfg.h_f * cfg.w_eff), device="cuda")
    out = torch.empty((n, cfg.c_out, h_out, w_out), device="cuda")
    im2win_into(x, win, cfg.params)
    conv_windows_into(win, f, out, cfg.params, cfg.w_eff)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        conv_windows_into(win, f, out, cfg.params, cfg.w_eff)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    tiles = -(-cfg.c_out // 64) * -(-n * h_out * w_out // 256)
    print(f"{name} N={n:4d} tiles={tiles:6d} waves={tiles / 296:6.2f} {best:8.3f} ms  {best / n * 1000:7.2f} us/img "
          f"{cfg.flops / best / 1e9:6.2f} TF", flush=True)
    del x, f, win, out
    torch.cuda.empty_cache()
