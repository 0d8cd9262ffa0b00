"""Direct TC kernel time per library build (exploration): python tools/direct_ab.py LIB... [--layers conv1,conv2]"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
if "--child" in sys.argv:
    sys.path.insert(0, str(ROOT))
    from dataclasses import replace

    import torch

    from paper_2306_14316_b200.kernels import conv_direct_into
    from paper_2306_14316_b200.workloads import BENCHMARKS

    dev = torch.device("cuda:0")
    out = []
    for name in sys.argv[sys.argv.index("--child") + 1].split(","):
        cfg = replace(BENCHMARKS[name], batch=128)
        h_out, w_out = cfg.out_dims
        x = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
        f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev)
        o = torch.empty((cfg.batch, cfg.c_out, h_out, w_out), device=dev)
        for v in ("tf32", "bf16"):
            conv_direct_into(x, f, o, cfg.params, v)
            torch.cuda.synchronize()
            ts = []
            for _ in range(15):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                conv_direct_into(x, f, o, cfg.params, v)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ts.sort()
            out.append(f"{name}/{v} {cfg.flops / ts[len(ts) // 2] / 1e9:7.1f}")
    print("RESULT " + " | ".join(out))
else:
    libs = [a for a in sys.argv[1:] if not a.startswith("--")]
    layers = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--layers=")), "conv1,conv2,conv3,conv7")
    for rnd in range(int(os.environ.get("AB_ROUNDS", "2"))):
        for lib in libs:
            env = dict(os.environ, IM2WIN_LIB=str(Path(lib).resolve()))
            r = subprocess.run([sys.executable, __file__, "--child", layers], env=env, capture_output=True, text=True)
            line = [x for x in r.stdout.splitlines() if x.startswith("RESULT")]
            print(f"{Path(lib).parent.name:10s}", line[0][7:] if line else r.stderr[-500:], flush=True)
