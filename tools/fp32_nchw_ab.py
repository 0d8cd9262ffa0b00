"""FP32-exact conv: transform + conv over Ĩ vs the same kernels gathering straight from NCHW.

    python tools/fp32_nchw_ab.py [layers|all] [batch]

Prints per layer: transform ms, conv-over-Ĩ ms, NCHW-direct conv ms, TFLOPS of (transform+conv)
and of the direct conv, and whether the two outputs are bit-identical.
"""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2306_14316_b200 as pkg  # noqa: E402
from paper_2306_14316_b200 import _lib  # noqa: E402
from paper_2306_14316_b200.kernels import conv_nchw_into, conv_windows_into  # noqa: E402
from paper_2306_14316_b200.layouts import im2win_into  # noqa: E402

layers = sys.argv[1].split(",") if len(sys.argv) > 1 and sys.argv[1] != "all" else list(pkg.BENCHMARKS)
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
dev = torch.device("cuda:0")


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best


print(f"{'layer':7s} {'xform':>7s} {'conv(Ĩ)':>8s} {'conv(X)':>8s} {'TF x+c':>7s} {'TF X':>7s} same kernel")
tot = [0.0, 0.0, 0.0, 0.0]
for name in layers:
    cfg = replace(pkg.BENCHMARKS[name], batch=batch)
    h_out, w_out = cfg.out_dims
    g = torch.Generator(device=dev).manual_seed(11)
    x = torch.randn((batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev, generator=g)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev, generator=g)
    win = torch.empty((batch, cfg.c_in, h_out, cfg.h_f * cfg.w_eff), device=dev)
    o1 = torch.empty((batch, cfg.c_out, h_out, w_out), device=dev)
    o2 = torch.full_like(o1, float("nan"))
    t_x = timed(lambda: im2win_into(x, win, cfg.params))
    t_c = timed(lambda: conv_windows_into(win, f, o1, cfg.params, cfg.w_eff))
    t_d = timed(lambda: conv_nchw_into(x, f, o2, cfg.params))
    kern = _lib.last_kernel()
    same = bool(torch.equal(o1.view(torch.int32), o2.view(torch.int32)))
    fl = cfg.flops
    tot[0] += t_x
    tot[1] += t_c
    tot[2] += t_d
    tot[3] += fl
    print(f"{name:7s} {t_x:7.3f} {t_c:8.3f} {t_d:8.3f} {fl / (t_x + t_c) / 1e9:7.1f} {fl / t_d / 1e9:7.1f} {same} {kern}",
          flush=True)
print(f"{'total':7s} {tot[0]:7.3f} {tot[1]:8.3f} {tot[2]:8.3f} {tot[3] / (tot[0] + tot[1]) / 1e9:7.1f} "
      f"{tot[3] / tot[2] / 1e9:7.1f}")
