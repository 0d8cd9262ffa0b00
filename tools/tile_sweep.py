"""Time every compiled SIMT CTA tile on a few layers (exploration; prints a table)."""
import ctypes
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_14316_b200 import _lib  # noqa: E402
from paper_2306_14316_b200.layouts import im2win_into  # noqa: E402
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

layers = sys.argv[1].split(",") if len(sys.argv) > 1 else ["conv4", "conv8", "conv9", "conv5", "conv6", "conv12", "conv1", "conv7"]
cfgs = range(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
import os  # noqa: E402
lib = _lib.load(os.environ.get("IM2WIN_LIB")) if os.environ.get("IM2WIN_LIB") else _lib.load()
dev = torch.device("cuda:0")
stream = torch.cuda.current_stream().cuda_stream
for name in layers:
    cfg = replace(BENCHMARKS[name], batch=128)
    h_out, w_out = cfg.out_dims
    x = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev)
    win = torch.empty((cfg.batch, cfg.c_in, h_out, cfg.h_f * cfg.w_eff), device=dev)
    ref = None
    im2win_into(x, win, cfg.params)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        im2win_into(x, win, cfg.params)
    e1.record()
    torch.cuda.synchronize()
    tr_ms = e0.elapsed_time(e1) / 3
    ws = torch.empty(lib.im2win_conv_workspace_bytes(cfg.c_in, cfg.c_out, cfg.h_f, cfg.w_f, 0), dtype=torch.uint8, device=dev)
    row = [f"{name:7s} tr {cfg.transform_bytes() / tr_ms / 1e6:7.0f} GB/s |"]
    for c in cfgs:
        out = torch.empty((cfg.batch, cfg.c_out, h_out, w_out), device=dev)
        plan = _lib.TilePlanC(c, 1, 1, 1)

        def run():
            rc = lib.im2win_conv_f32(win.data_ptr(), f.data_ptr(), out.data_ptr(), cfg.batch, cfg.c_in, cfg.c_out,
                                     h_out, w_out, cfg.h_f * cfg.w_eff, cfg.h_f, cfg.w_f, cfg.stride,
                                     ctypes.byref(plan), 0, ws.data_ptr(), ws.numel(), stream)
            _lib.check(rc)
        run()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            e0.record()
            for _ in range(5):
                run()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 5)
        if ref is None:
            ref = out.clone()
        same = torch.equal(out.view(torch.int32), ref.view(torch.int32))
        row.append(f" c{c} {cfg.flops / best / 1e9:6.1f}{'' if same else '!'}")
    print("".join(row), flush=True)
