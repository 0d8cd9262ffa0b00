"""Fused TC conv time per library build, through the symbols every round's library exports
(im2win_nchw_to_nhwc + im2win_conv_fused), so builds from earlier commits compare too:

    python tools/tc_conv_ab.py LIB... [--layers=conv5,conv12] [--batch=128] [--variants=tf32,bf16]

Prints TFLOPS of the copy + conv and of the conv alone; rounds alternate between libraries.
"""
import ctypes
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def child(lib_path, layers, batch, variants):
    sys.path.insert(0, str(ROOT))
    from dataclasses import replace

    import torch

    from paper_2306_14316_b200.workloads import BENCHMARKS

    lib = ctypes.CDLL(lib_path)
    i64, i32, vp, sz = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t
    lib.im2win_nchw_to_nhwc.argtypes = [vp, vp, i64, i64, i64, i64, i32, vp]
    lib.im2win_conv_fused_workspace_bytes.argtypes = [i64, i64, i32, i32]
    lib.im2win_conv_fused_workspace_bytes.restype = sz
    lib.im2win_conv_fused.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i32, i32, i32, i32, vp, sz, vp]
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream().cuda_stream
    out = []
    for name in layers:
        cfg = replace(BENCHMARKS[name], batch=batch)
        h_out, w_out = cfg.out_dims
        x = torch.randn((batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
        f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev)
        o = torch.empty((batch, cfg.c_out, h_out, w_out), device=dev)
        for v in variants:
            bf = v == "bf16"
            pitch = -(-cfg.c_in // (8 if bf else 4)) * (8 if bf else 4)
            xc = torch.empty((batch, cfg.h_in, cfg.w_in, pitch), device=dev,
                             dtype=torch.bfloat16 if bf else torch.float32)
            nb = lib.im2win_conv_fused_workspace_bytes(cfg.c_in, cfg.c_out, cfg.h_f, cfg.w_f)
            ws = torch.empty(nb, dtype=torch.uint8, device=dev)

            def cp():
                assert lib.im2win_nchw_to_nhwc(x.data_ptr(), xc.data_ptr(), batch, cfg.c_in, cfg.h_in, cfg.w_in,
                                               1 if bf else 0, st) == 0

            def cv():
                assert lib.im2win_conv_fused(xc.data_ptr(), f.data_ptr(), o.data_ptr(), batch, cfg.c_in, cfg.h_in,
                                             cfg.w_in, cfg.c_out, cfg.h_f, cfg.w_f, cfg.stride, 3 if bf else 2,
                                             ws.data_ptr(), nb, st) == 0

            res = []
            for fns in ((cp, cv), (cv,)):
                for fn in fns:
                    fn()
                torch.cuda.synchronize()
                ts = []
                for _ in range(9):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    for fn in fns:
                        fn()
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b))
                ts.sort()
                res.append(cfg.flops / ts[len(ts) // 2] / 1e9)
            out.append(f"{name}/{v} {res[0]:6.1f} {res[1]:6.1f}")
    print("RESULT " + " | ".join(out))


if __name__ == "__main__":
    opts = {a.split("=", 1)[0]: a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--") and "=" in a}
    layers = opts.get("--layers", "conv5,conv6,conv11,conv12").split(",")
    batch = int(opts.get("--batch", "128"))
    variants = opts.get("--variants", "tf32,bf16").split(",")
    if "--child" in sys.argv:
        child(opts["--lib"], layers, batch, variants)
        sys.exit(0)
    libs = [a for a in sys.argv[1:] if not a.startswith("--")]
    for rnd in range(int(os.environ.get("AB_ROUNDS", "2"))):
        for lib in libs:
            r = subprocess.run([sys.executable, __file__, "--child", f"--lib={Path(lib).resolve()}"]
                               + [a for a in sys.argv[1:] if a.startswith("--")], capture_output=True, text=True)
            line = [x for x in r.stdout.splitlines() if x.startswith("RESULT")]
            print(f"{Path(lib).parent.name:8s}", line[0][7:] if line else r.stderr[-400:], flush=True)
