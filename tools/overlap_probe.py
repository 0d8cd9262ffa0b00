"""Does the channels-last copy of image chunk k+1 overlap the fused TC conv of chunk k?
(exploration: the copy is HBM-bound, the conv kernels smem/tensor-bound).

    python tools/overlap_probe.py [layers] [chunks...]
"""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_14316_b200.kernels import conv_fused_into, nhwc_into, nhwc_pitch  # noqa: E402
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

layers = sys.argv[1].split(",") if len(sys.argv) > 1 else ["conv4", "conv8", "conv5"]
chunk_counts = [int(c) for c in sys.argv[2:]] or [2, 4, 8]
dev = torch.device("cuda:0")
main = torch.cuda.current_stream(dev)
side = torch.cuda.Stream(dev)


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        fn()
        b.record(main)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


for name in layers:
    cfg = replace(BENCHMARKS[name], batch=128)
    h_out, w_out = cfg.out_dims
    x = torch.randn((128, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev)
    out = torch.empty((128, cfg.c_out, h_out, w_out), device=dev)
    for variant in ("bf16", "tf32"):
        dt = torch.bfloat16 if variant == "bf16" else torch.float32
        xcl = torch.empty((128, cfg.h_in, cfg.w_in, nhwc_pitch(cfg.c_in, variant)), dtype=dt, device=dev)

        def whole():
            nhwc_into(x, xcl)
            conv_fused_into(xcl, f, out, cfg.params, variant)

        ref = None
        whole()
        ref = out.clone()
        row = [f"{name:6s} {variant}: whole {timed(whole):.3f} ms"]
        row.append(f"(copy {timed(lambda: nhwc_into(x, xcl)):.3f}, conv {timed(lambda: conv_fused_into(xcl, f, out, cfg.params, variant)):.3f})")
        for nc in chunk_counts:
            c = 128 // nc

            def chunked():
                evs = []
                side.wait_stream(main)
                with torch.cuda.stream(side):
                    for k in range(nc):
                        nhwc_into(x[k * c:(k + 1) * c], xcl[k * c:(k + 1) * c])
                        e = torch.cuda.Event()
                        e.record(side)
                        evs.append(e)
                for k in range(nc):
                    main.wait_event(evs[k])
                    conv_fused_into(xcl[k * c:(k + 1) * c], f, out[k * c:(k + 1) * c], cfg.params, variant)

            t = timed(chunked)
            same = torch.equal(out, ref)
            row.append(f"| {nc} chunks {t:.3f}{'' if same else ' MISMATCH'}")
        print(" ".join(row), flush=True)
