"""Small invocations of every kernel family, for compute-sanitizer runs:

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
    compute-sanitizer --tool synccheck python tools/sanitize_cases.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_14316_b200 as pkg  # noqa: E402

rng = np.random.default_rng(0)
cases = [(2, 3, 13, 15, 16, 3, 3, 1, 0), (1, 8, 11, 9, 8, 5, 5, 2, 1), (2, 16, 10, 10, 32, 3, 3, 1, 1),
         (1, 4, 23, 23, 96, 11, 11, 4, 0), (1, 64, 12, 12, 64, 7, 7, 2, 3)]
for (n, c, h, w, co, hf, wf, s, p) in cases:
    x = torch.from_numpy(rng.standard_normal((n, c, h, w), dtype=np.float32)).cuda()
    f = torch.from_numpy(rng.standard_normal((co, c, hf, wf), dtype=np.float32)).cuda()
    params = pkg.ConvParams(c, co, hf, wf, s, pad=p)
    pkg.conv_im2win_opt(x, f, params)
    pkg.conv_im2win_opt(x, f, params, variant="fp32-fma")
    win = pkg.im2win(x, params)
    pkg.compute_from_windows_basic(win, f, params)
    pkg.compute_from_windows_opt(win, f, params, pkg.TilePlan(64, 64, 8, 4, 4))
    for v in ("tf32", "bf16"):
        for path in ("fused", "gather", "direct"):
            if path == "direct" and not pkg.kernels.direct_supported(x.shape, params, v):
                continue
            pkg.conv_im2win_opt(x, f, params, variant=v, tc_path=path)
    pkg.conv_im2win_opt_host(x.cpu(), f.cpu(), params, chunk_images=1)
# round 2: the in-kernel channels-last feed (forced on every TMA-fed kernel), CTA pairs, tap pairs
# in the phase kernel (smem exchange between epilogue warps), the FP32 window-budget chunks
import os  # noqa: E402

for (n, c, h, w, co, hf, wf, s, p) in cases:
    if p:
        continue
    x = torch.from_numpy(rng.standard_normal((n + 2, c, h, w), dtype=np.float32)).cuda()
    f = torch.from_numpy(rng.standard_normal((co, c, hf, wf), dtype=np.float32)).cuda()
    params = pkg.ConvParams(c, co, hf, wf, s)
    for env in ({"IM2WIN_FEED": "2"}, {"IM2WIN_FEED": "2", "IM2WIN_FEED_ROUNDS": "1"},
                {"IM2WIN_FEED": "2", "IM2WIN_PAIR": "1", "IM2WIN_PHASE": "2"}):
        os.environ.update(env)
        for v in ("tf32", "bf16"):
            pkg.conv_im2win_opt(x, f, params, variant=v, tc_path="fused")
        for k in env:
            del os.environ[k]
    os.environ["IM2WIN_WINDOW_BUDGET"] = "1"
    pkg.conv_im2win_opt(torch.cat([x] * 5), f, params)
    del os.environ["IM2WIN_WINDOW_BUDGET"]
# shapes the phase kernel takes (C >= 32, stride <= 2, Co <= 64): tap pairs with and without the feed
for (n, c, h, w, co, hf, wf, s) in [(2, 64, 17, 19, 64, 7, 7, 2), (3, 32, 9, 10, 48, 3, 3, 1)]:
    x = torch.from_numpy(rng.standard_normal((n, c, h, w), dtype=np.float32)).cuda()
    f = torch.from_numpy(rng.standard_normal((co, c, hf, wf), dtype=np.float32)).cuda()
    params = pkg.ConvParams(c, co, hf, wf, s)
    for env in ({"IM2WIN_PHASE": "2", "IM2WIN_PHASE_TN2": "2"},
                {"IM2WIN_FEED": "2", "IM2WIN_PHASE": "2", "IM2WIN_PHASE_TN2": "2"},
                {"IM2WIN_PAIR": "1", "IM2WIN_PHASE": "2", "IM2WIN_PHASE_TN2": "2"}):
        os.environ.update(env)
        for v in ("tf32", "bf16"):
            pkg.conv_im2win_opt(x, f, params, variant=v, tc_path="fused")
            assert "tap pairs" in pkg._lib.last_kernel(), pkg._lib.last_kernel()
        for k in env:
            del os.environ[k]
# a 96-channel layer big enough for the library's 64 + 32 channel split (packed exact MACs)
x = torch.from_numpy(rng.standard_normal((32, 3, 131, 131), dtype=np.float32)).cuda()
f = torch.from_numpy(rng.standard_normal((96, 3, 11, 11), dtype=np.float32)).cuda()
pkg.conv_im2win_opt(x, f, pkg.ConvParams(3, 96, 11, 11, 4))
assert "64-95" in pkg._lib.last_kernel(), pkg._lib.last_kernel()
# 4-byte-offset operands (the staged transform aligns its 16-byte copies to the address)
for (n, c, h, w, co, hf, wf, s, p) in cases[:3]:
    base = torch.from_numpy(rng.standard_normal(1 + n * c * h * w, dtype=np.float32)).cuda()
    x = base[1:].view(n, c, h, w)
    f = torch.from_numpy(rng.standard_normal((co, c, hf, wf), dtype=np.float32)).cuda()
    params = pkg.ConvParams(c, co, hf, wf, s, pad=p)
    pkg.conv_im2win_opt(x, f, params)
    pkg.im2win(x, params)
torch.cuda.synchronize()
print("sanitize cases done")
