import sys, time
sys.path.insert(0, "/root/repo")
from dataclasses import replace
import torch
import paper_2306_14316_b200 as pkg
from paper_2306_14316_b200.kernels import conv_fused_nchw_into, conv_nchw_into, nhwc_pitch
dev = torch.device("cuda:0")
for name, v in (("conv12", "bf16"), ("conv11", "bf16"), ("conv12", "fp32-exact")):
    cfg = replace(pkg.BENCHMARKS[name], batch=128)
    x = torch.randn((128, cfg.c_in, cfg.h_in, cfg.w_in), device=dev)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=dev)
    h_out, w_out = cfg.out_dims
    o = torch.empty((128, cfg.c_out, h_out, w_out), device=dev)
    if v == "fp32-exact":
        call = lambda: conv_nchw_into(x, f, o, cfg.params)
    else:
        xc = torch.empty((128, cfg.h_in, cfg.w_in, nhwc_pitch(cfg.c_in, v)), device=dev, dtype=torch.bfloat16)
        call = lambda: conv_fused_nchw_into(x, xc, f, o, cfg.params, v)
    call(); torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        call()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        call()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        call()
    g.replay(); torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        g.replay()
    b.record(); torch.cuda.synchronize()
    print(f"{name} {v}: host enqueue {1e6*(t1-t0)/n:.1f} us/call, wall {1e6*(t2-t0)/n:.1f} us/call, graph-replay GPU {1e3*a.elapsed_time(b)/n:.1f} us/call")
