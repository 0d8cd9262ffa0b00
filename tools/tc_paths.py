"""Compare the tensor-core paths (fused / cl / gather): parity at batch 2 and speed at batch N."""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2306_14316_b200 as pkg  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2306_14316_b200.kernels import conv_fused_into, nhwc_into, nhwc_pitch  # noqa: E402

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
    cfg = pkg.BENCHMARKS[name]
    for v in ("tf32", "bf16"):
        c2 = replace(cfg, batch=2, seed=9)
        inp, flt = pkg.make_inputs(c2)
        ref = orc.conv_direct(inp, flt, c2.stride)
        errs = {p: pkg.normalized_max_diff(pkg.conv_im2win_opt(inp, flt, c2.params, variant=v, tc_path=p).numpy(), ref)
                for p in ("fused", "cl")}
        cb = replace(cfg, batch=batch)
        x = torch.randn((cb.batch, cb.c_in, cb.h_in, cb.w_in), device=dev)
        f = torch.randn((cb.c_out, cb.c_in, cb.h_f, cb.w_f), device=dev)
        h_out, w_out = cb.out_dims
        o = torch.empty((cb.batch, cb.c_out, h_out, w_out), device=dev)
        xc = torch.empty((cb.batch, cb.h_in, cb.w_in, nhwc_pitch(cb.c_in, v)), device=dev,
                         dtype=torch.bfloat16 if v == "bf16" else torch.float32)
        t_tr = timed(lambda: nhwc_into(x, xc))
        t_cv = timed(lambda: conv_fused_into(xc, f, o, cb.params, v))
        t_cl = timed(lambda: pkg.conv_im2win_opt(x, f, cb.params, variant=v, tc_path="cl"))
        tr_bytes = 4 * x.numel() + xc.numel() * xc.element_size()
        print(f"{name:7s} {v} err fused {errs['fused']:.2e} cl {errs['cl']:.2e} | nhwc {tr_bytes / t_tr / 1e6:6.0f} GB/s "
              f"{t_tr:6.3f} ms | fused conv {cb.flops / t_cv / 1e9:7.1f} TF | fused total {cb.flops / (t_tr + t_cv) / 1e9:7.1f} TF"
              f" | cl total (api) {cb.flops / t_cl / 1e9:7.1f} TF", flush=True)
        del x, f, o, xc
        torch.cuda.empty_cache()
