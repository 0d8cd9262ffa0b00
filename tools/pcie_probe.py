"""Host<->device copy bandwidth on this box (pinned buffers): H2D, D2H, both at once.

The bound for bench.py's e2e number: every step moves its inputs up and its outputs down.
"""
import json
import sys

import torch

nbytes = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1 << 30
dev = torch.device("cuda:0")
h_src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
h_dst = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
d_a = torch.empty(nbytes, dtype=torch.uint8, device=dev)
d_b = torch.empty(nbytes, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best * 1e-3


def h2d():
    d_a.copy_(h_src, non_blocking=True)


def d2h():
    h_dst.copy_(d_b, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_src, non_blocking=True)
    with torch.cuda.stream(s2):
        h_dst.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"bytes": nbytes, "h2d_gbs": nbytes / t1 / 1e9, "d2h_gbs": nbytes / t2 / 1e9,
                  "bidir_each_gbs": nbytes / t3 / 1e9}))
