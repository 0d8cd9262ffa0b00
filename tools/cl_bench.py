"""Channels-innermost TC path: parity (normalized error vs oracle at batch 2) and per-layer speed at N."""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2306_14316_b200 as pkg  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2306_14316_b200.kernels import cl_supported, conv_cl_into, im2win_cl_into, im2win_cl_shape  # noqa: E402

layers = sys.argv[1].split(",") if len(sys.argv) > 1 and sys.argv[1] != "all" else list(pkg.BENCHMARKS)
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
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


for name in layers:
    for v in ("tf32", "bf16"):
        cfg = pkg.BENCHMARKS[name]
        if not cl_supported(cfg.c_in, v):
            continue
        c2 = replace(cfg, batch=2, seed=9)
        inp, flt = pkg.make_inputs(c2)
        out = pkg.conv_im2win_opt(inp, flt, c2.params, variant=v).numpy()
        err = pkg.normalized_max_diff(out, orc.conv_direct(inp, flt, c2.stride))
        cb = replace(cfg, batch=batch)
        h_out, w_out = cb.out_dims
        x = torch.randn((cb.batch, cb.c_in, cb.h_in, cb.w_in), device=dev)
        f = torch.randn((cb.c_out, cb.c_in, cb.h_f, cb.w_f), device=dev)
        wcl = torch.empty(im2win_cl_shape((cb.batch, cb.c_in, cb.h_in, cb.w_in), cb.params),
                          dtype=torch.bfloat16 if v == "bf16" else torch.float32, device=dev)
        o = torch.empty((cb.batch, cb.c_out, h_out, w_out), device=dev)
        t_tr = timed(lambda: im2win_cl_into(x, wcl, cb.params))
        t_cv = timed(lambda: conv_cl_into(wcl, f, o, cb.params, v))
        tr_bytes = 4 * cb.elems("raw") + wcl.numel() * wcl.element_size()
        print(f"{name:7s} {v} err {err:.2e} | transform_cl {tr_bytes / t_tr / 1e6:6.0f} GB/s {t_tr:7.3f} ms | "
              f"conv {cb.flops / t_cv / 1e9:7.1f} TF {t_cv:7.3f} ms | total {cb.flops / (t_tr + t_cv) / 1e9:7.1f} TF",
              flush=True)
        del x, f, wcl, o
        torch.cuda.empty_cache()
