"""Quick TF32/BF16 tensor-core parity check vs the oracle (normalized error)."""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_14316_b200 as pkg  # noqa: E402
from oracle import oracle as orc  # noqa: E402

layers = sys.argv[1].split(",") if len(sys.argv) > 1 else ["conv9"]
for name in layers:
    cfg = replace(pkg.BENCHMARKS[name], batch=2, seed=5)
    inp, flt = pkg.make_inputs(cfg)
    ref = orc.conv_direct(inp, flt, cfg.stride)
    for v in ("tf32", "bf16"):
        out = pkg.conv_im2win_opt(inp, flt, cfg.params, variant=v)
        torch.cuda.synchronize()
        o = out.numpy()
        print(name, v, "normalized", pkg.normalized_max_diff(o, ref), "max_rel", pkg.max_rel_diff(o, ref),
              "nan", int(np.isnan(o).sum()), flush=True)
