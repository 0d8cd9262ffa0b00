"""Per-layer time of every variant + cuDNN at N=128 (exploration / evidence table)."""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2306_14316_b200.kernels import conv_windows_into  # noqa: E402
from paper_2306_14316_b200.layouts import im2win_into  # noqa: E402
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

layers = sys.argv[1].split(",") if len(sys.argv) > 1 and sys.argv[1] != "all" else list(BENCHMARKS)
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
variants = ["fp32-exact", "fp32-fma", "tf32", "bf16"]
dev = torch.device("cuda:0")


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


print(f"{'layer':7s} {'tr GB/s':>8s} " + " ".join(f"{v:>10s}" for v in variants) +
      f" {'cudnn32':>8s} {'cudnnTF32':>9s} {'cudnnBF16':>9s}   (TFLOPS, conv only)", flush=True)
for name in layers:
    cfg = replace(BENCHMARKS[name], batch=batch)
    h_out, w_out = cfg.out_dims
    x = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev)
    win = torch.empty((cfg.batch, cfg.c_in, h_out, cfg.h_f * cfg.w_eff), device=dev)
    out = torch.empty((cfg.batch, cfg.c_out, h_out, w_out), device=dev)
    t_tr = timed(lambda: im2win_into(x, win, cfg.params))
    row = [f"{name:7s} {cfg.transform_bytes() / t_tr / 1e6:8.0f}"]
    for v in variants:
        t = timed(lambda: conv_windows_into(win, f, out, cfg.params, cfg.w_eff, None, v))
        row.append(f"{cfg.flops / t / 1e9:10.1f}")
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.allow_tf32 = False
    row.append(f"{cfg.flops / timed(lambda: F.conv2d(x, f, stride=cfg.stride)) / 1e9:8.1f}")
    torch.backends.cudnn.allow_tf32 = True
    row.append(f"{cfg.flops / timed(lambda: F.conv2d(x, f, stride=cfg.stride)) / 1e9:9.1f}")
    xb, fb = x.bfloat16(), f.bfloat16()
    row.append(f"{cfg.flops / timed(lambda: F.conv2d(xb, fb, stride=cfg.stride)) / 1e9:9.1f}")
    torch.backends.cudnn.allow_tf32 = False
    print(" ".join(row), flush=True)
    del x, f, win, out
    torch.cuda.empty_cache()
