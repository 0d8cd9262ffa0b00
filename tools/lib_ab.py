"""Production-path time per library build (exploration A/B of build flags):

    python tools/lib_ab.py LIB... [--layers=conv3,conv7] [--batch=128] [--variants=tf32,bf16]

Each library runs in its own process (IM2WIN_LIB); rounds alternate between libraries
(AB_ROUNDS, default 2) so box drift shows up as round-to-round spread, not as a difference.
"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def child(layers, batch, variants):
    sys.path.insert(0, str(ROOT))
    from dataclasses import replace

    import torch

    import paper_2306_14316_b200 as pkg
    from paper_2306_14316_b200.workloads import BENCHMARKS

    dev = torch.device("cuda:0")
    out = []
    for name in layers:
        cfg = replace(BENCHMARKS[name], batch=batch)
        x = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
        f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev)
        for v in variants:
            pkg.conv_im2win_opt(x, f, cfg.params, variant=v)
            torch.cuda.synchronize()
            ts = []
            for _ in range(9):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                pkg.conv_im2win_opt(x, f, cfg.params, variant=v)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ts.sort()
            out.append(f"{name}/{v} {cfg.flops / ts[len(ts) // 2] / 1e9:7.1f}")
    print("RESULT " + " | ".join(out))


if __name__ == "__main__":
    opts = {a.split("=", 1)[0]: a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--") and "=" in a}
    layers = opts.get("--layers", "conv3,conv7,conv8,conv9").split(",")
    batch = int(opts.get("--batch", "128"))
    variants = opts.get("--variants", "tf32,bf16").split(",")
    if "--child" in sys.argv:
        child(layers, batch, variants)
        sys.exit(0)
    libs = [a for a in sys.argv[1:] if not a.startswith("--")]
    for rnd in range(int(os.environ.get("AB_ROUNDS", "2"))):
        for lib in libs:
            env = dict(os.environ, IM2WIN_LIB=str(Path(lib).resolve()))
            r = subprocess.run([sys.executable, __file__, "--child"] + [a for a in sys.argv[1:] if a.startswith("--")],
                               env=env, capture_output=True, text=True)
            line = [x for x in r.stdout.splitlines() if x.startswith("RESULT")]
            print(f"{Path(lib).parent.name:8s}", line[0][7:] if line else r.stderr[-400:], flush=True)
