"""im2win transform: bit-exactness against a torch unfold restatement and GB/s per layer.

    python tools/transform_bench.py [layers|all] [batch] [chunk targets, comma list]

Chunk target (floats of output per chunk) is passed through IM2WIN_XFORM_CHUNK.
"""
import os
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_14316_b200.layouts import im2win_into  # noqa: E402
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

layers = sys.argv[1].split(",") if len(sys.argv) > 1 and sys.argv[1] != "all" else list(BENCHMARKS)
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
targets = [int(t) for t in sys.argv[3].split(",")] if len(sys.argv) > 3 else [4096]
peak = 6536.0
dev = torch.device("cuda:0")
tot_b = {t: 0.0 for t in targets}
tot_t = {t: 0.0 for t in targets}
for name in layers:
    cfg = replace(BENCHMARKS[name], batch=batch)
    h_out, w_out = cfg.out_dims
    x = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
    win = torch.empty((cfg.batch, cfg.c_in, h_out, cfg.h_f * cfg.w_eff), device=dev)
    ref = x.unfold(2, cfg.h_f, cfg.stride)[:, :, :h_out, :cfg.w_eff, :].reshape(win.shape)
    row = [f"{name:7s}"]
    for t in targets:
        os.environ["IM2WIN_XFORM_CHUNK"] = str(t)
        win.fill_(float("nan"))
        im2win_into(x, win, cfg.params)
        torch.cuda.synchronize()
        ok = bool(torch.equal(win.view(torch.int32), ref.contiguous().view(torch.int32)))
        best = 1e30
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            im2win_into(x, win, cfg.params)
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        gbs = cfg.transform_bytes() / (best * 1e-3) / 1e9
        tot_b[t] += cfg.transform_bytes()
        tot_t[t] += best * 1e-3
        row.append(f"t={t:6d} {best * 1e3:8.1f}us {gbs:7.0f}GB/s {gbs / peak:5.1%} {'ok' if ok else 'MISMATCH'}")
    print("  ".join(row), flush=True)
    del x, win, ref
    torch.cuda.empty_cache()
for t in targets:
    print(f"all t={t}: {tot_b[t] / tot_t[t] / 1e9:.0f} GB/s ({tot_b[t] / tot_t[t] / 1e9 / peak:.1%})")
