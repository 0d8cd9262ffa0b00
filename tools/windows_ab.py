"""Few-channel tensor-core layers: channels-last copy + conv vs window image + 1x1 conv vs the direct kernel.

    python tools/windows_ab.py [layers] [batch] [variants]

The one-call entry (im2win_conv_fused_nchw) is timed with IM2WIN_WINDOWS=0 (channels-last copy,
then the fused/shift/phase kernel) and 2 (window image, then the 1x1 conv); the direct kernel
through im2win_conv_direct.  Error = max|d| / rms(ref) against the FP32-exact production call.
"""
import os
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_14316_b200 import _lib  # noqa: E402
from paper_2306_14316_b200.kernels import conv_fused_nchw_into, conv_nchw_into, nhwc_pitch  # noqa: E402
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

layers = (sys.argv[1] if len(sys.argv) > 1 else "conv1,conv2,conv3,conv7").split(",")
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
variants = (sys.argv[3] if len(sys.argv) > 3 else "bf16,tf32").split(",")
dev = torch.device("cuda:0")


def timed(fn, reps=7):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def err(o, ref):
    return float((o - ref).abs().max() / ref.pow(2).mean().sqrt())


for name in layers:
    cfg = replace(BENCHMARKS[name], batch=batch)
    h_out, w_out = cfg.out_dims
    g = torch.Generator(device=dev).manual_seed(9)
    x = torch.randn((batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev, generator=g)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev, generator=g)
    ref = torch.empty((batch, cfg.c_out, h_out, w_out), device=dev)
    conv_nchw_into(x, f, ref, cfg.params)
    out = torch.empty_like(ref)
    k = cfg.c_in * cfg.h_f * cfg.w_f
    for v in variants:
        bf = v == "bf16"
        esz = 2 if bf else 4
        nb = max(batch * cfg.h_in * cfg.w_in * nhwc_pitch(cfg.c_in, v), batch * h_out * w_out * nhwc_pitch(k, v)) * esz
        scratch = torch.empty(nb, dtype=torch.uint8, device=dev)
        row = []
        for mode in ("0", "2"):
            os.environ["IM2WIN_WINDOWS"] = mode
            out.fill_(float("nan"))
            t = timed(lambda: conv_fused_nchw_into(x, scratch, f, out, cfg.params, v))
            row.append(f"{'copy' if mode == '0' else 'windows'} {t:7.3f} ms {cfg.flops / t / 1e9:6.1f} TF "
                       f"err {err(out, ref):.1e} [{_lib.last_kernel()}]")
        os.environ["IM2WIN_WINDOWS"] = "0"
        lib = _lib.load()
        code = 3 if bf else 2
        if lib.im2win_conv_direct_supported(batch, cfg.c_in, cfg.h_in, cfg.w_in, cfg.c_out, cfg.h_f, cfg.w_f,
                                            cfg.stride, 0, code):
            wsb = lib.im2win_conv_direct_workspace(cfg.c_in, cfg.c_out, cfg.h_f, cfg.w_f, code)
            ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
            st = torch.cuda.current_stream().cuda_stream

            def direct():
                _lib.check(lib.im2win_conv_direct(x.data_ptr(), f.data_ptr(), out.data_ptr(), batch, cfg.c_in,
                                                  cfg.h_in, cfg.w_in, cfg.c_out, cfg.h_f, cfg.w_f, cfg.stride, 0,
                                                  code, ws.data_ptr(), wsb, st))
            out.fill_(float("nan"))
            t = timed(direct)
            row.append(f"direct {t:7.3f} ms {cfg.flops / t / 1e9:6.1f} TF err {err(out, ref):.1e}")
        print(f"{name:6s} {v:5s} N={batch} | " + " | ".join(row), flush=True)
        del scratch
