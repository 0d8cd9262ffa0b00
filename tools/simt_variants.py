"""FP32 conv-only time of every benchmark layer for several library builds (exploration).

    python tools/simt_variants.py build/var_a/libim2win_sm100.so build/var_b/libim2win_sm100.so ...

Each build runs in its own subprocess (IM2WIN_LIB) on the same seeded inputs; the
script prints per-layer TFLOPS and the 12-layer total, and checks every build's
output bits against the first one.
"""
import json
import os
import subprocess
import sys
from dataclasses import replace
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def child(batch: int, variant: str, reps: int) -> None:
    import hashlib

    import torch

    from paper_2306_14316_b200.kernels import conv_windows_into
    from paper_2306_14316_b200.layouts import im2win_into
    from paper_2306_14316_b200.workloads import BENCHMARKS

    dev = torch.device("cuda:0")
    res = {}
    for name, cfg in BENCHMARKS.items():
        cfg = replace(cfg, batch=batch)
        h_out, w_out = cfg.out_dims
        g = torch.Generator(device=dev).manual_seed(7)
        x = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev, generator=g)
        f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev, generator=g)
        win = torch.empty((cfg.batch, cfg.c_in, h_out, cfg.h_f * cfg.w_eff), device=dev)
        out = torch.empty((cfg.batch, cfg.c_out, h_out, w_out), device=dev)
        im2win_into(x, win, cfg.params)
        fn = lambda: conv_windows_into(win, f, out, cfg.params, cfg.w_eff, None, variant)  # noqa: E731
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
        digest = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16]
        res[name] = {"ms": ts[len(ts) // 2], "gflop": cfg.flops / 1e9, "sha": digest}
        del x, f, win, out
        torch.cuda.empty_cache()
    print("RESULT " + json.dumps(res), flush=True)


def main() -> None:
    libs = [a for a in sys.argv[1:] if not a.startswith("--")]
    opts = dict(a[2:].split("=", 1) for a in sys.argv[1:] if a.startswith("--"))
    batch, variant, reps = int(opts.get("batch", 128)), opts.get("variant", "fp32-exact"), int(opts.get("reps", 7))
    table = {}
    for lib in libs:
        env = dict(os.environ, IM2WIN_LIB=str(Path(lib).resolve()))
        r = subprocess.run([sys.executable, __file__, "--child", f"--batch={batch}", f"--variant={variant}",
                            f"--reps={reps}"], env=env, capture_output=True, text=True)
        line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
        if not line:
            print(lib, "FAILED", r.stderr[-2000:])
            continue
        table[lib] = json.loads(line[0][7:])
    if not table:
        return
    names = list(next(iter(table.values())))
    first = next(iter(table.values()))
    print(f"{'layer':7s} " + " ".join(f"{Path(lib).parent.name[-14:]:>14s}" for lib in table))
    for n in names:
        print(f"{n:7s} " + " ".join(
            f"{t[n]['gflop'] / t[n]['ms']:12.2f}{'  ' if t[n]['sha'] == first[n]['sha'] else ' !'}"
            for t in table.values()))
    print(f"{'total':7s} " + " ".join(
        f"{sum(t[n]['gflop'] for n in names) / sum(t[n]['ms'] for n in names):12.2f}  " for t in table.values()))


if __name__ == "__main__":
    if "--child" in sys.argv:
        o = dict(a[2:].split("=", 1) for a in sys.argv[1:] if a.startswith("--") and "=" in a)
        child(int(o["batch"]), o["variant"], int(o["reps"]))
    else:
        main()
