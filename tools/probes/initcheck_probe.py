import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2306_14316_b200 as pkg
from paper_2306_14316_b200.layouts import im2win_into
from paper_2306_14316_b200.kernels import conv_windows_into
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.standard_normal((2, 3, 13, 15), dtype=np.float32)).cuda()
f = torch.from_numpy(rng.standard_normal((16, 3, 3, 3), dtype=np.float32)).cuda()
p = pkg.ConvParams(3, 16, 3, 3, 1)
mode = sys.argv[1]
win = (torch.zeros if mode == "zeros" else torch.empty)((2, 3, 11, 3 * 15), device="cuda")
out = torch.empty((2, 16, 11, 13), device="cuda")
im2win_into(x, win, p)
conv_windows_into(win, f, out, p, 15)
torch.cuda.synchronize()
print("done", mode)
