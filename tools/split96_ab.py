import os, sys
sys.path.insert(0, "/root/repo")
from dataclasses import replace
import torch
import paper_2306_14316_b200 as pkg
from paper_2306_14316_b200 import _lib
from paper_2306_14316_b200.kernels import conv_nchw_into
dev = torch.device("cuda:0")
for name in ("conv1", "conv2"):
    cfg = replace(pkg.BENCHMARKS[name], batch=128)
    x = torch.randn((128, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev)
    outs = []
    for mode in ("0", "1"):
        os.environ["IM2WIN_SIMT_SPLIT96"] = mode
        o = torch.empty((128, cfg.c_out) + cfg.out_dims, device=dev)
        conv_nchw_into(x, f, o, cfg.params); torch.cuda.synchronize()
        ts = []
        for _ in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); conv_nchw_into(x, f, o, cfg.params); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        t = sorted(ts)[3]
        outs.append(o)
        print(name, "split" if mode == "1" else "96x128", f"{t:.3f} ms {cfg.flops / t / 1e9:.1f} TF", _lib.last_kernel())
    print(name, "bit-identical:", torch.equal(outs[0].view(torch.int32), outs[1].view(torch.int32)))
