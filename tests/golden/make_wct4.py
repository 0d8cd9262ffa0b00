"""Generate WCT4 fixtures WITH THE REFERENCE ITSELF (its `winconv` CLI), for the interchange tests.

The reference CLI reads an input fixture, writes the im2win transform (`winconv transform
--layout im2win`, /root/reference/pkg/src/winconv/cli.py:137-149) and the convolution output
(`winconv conv --algo im2win-opt`, cli.py:152-174) as WCT4 files (fixture_io.py:25-66).  The
inputs themselves are written here with numpy (the format is a 40-byte header + row-major
float32), and the reference reads them back.  Run in the build container (the reference is
at /root/reference; it is absent on the GPU box, so the outputs are committed):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_wct4.py
"""

import os
import struct
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent / "wct4"
REF = Path("/root/reference/pkg/src")

# (name, input dims, filter dims, stride, seed)
CASES = [
    ("fig1", (1, 3, 3, 4), (2, 3, 2, 2), 1, 0),
    ("ragged", (2, 5, 9, 11), (4, 5, 3, 3), 1, 1),
    ("strided", (1, 3, 23, 21), (6, 3, 5, 5), 2, 2),
    ("special", (1, 2, 6, 7), (3, 2, 2, 3), 1, 3),
]


def write_wct4(arr: np.ndarray, path: Path) -> None:
    a = np.ascontiguousarray(arr, dtype=np.float32)
    with open(path, "wb") as fh:
        fh.write(b"WCT4")
        fh.write(struct.pack("<I", 1))
        fh.write(struct.pack("<4Q", *a.shape))
        fh.write(a.tobytes(order="C"))


def main() -> None:
    HERE.mkdir(exist_ok=True)
    env = dict(os.environ, PYTHONPATH=str(REF), NUMBA_CACHE_DIR=os.environ.get("NUMBA_CACHE_DIR", "/tmp/numba_cache"))
    for name, idims, fdims, stride, seed in CASES:
        rng = np.random.default_rng(seed)
        if name == "fig1":
            x = np.arange(1, np.prod(idims) + 1, dtype=np.float32).reshape(idims)
        else:
            x = rng.standard_normal(idims, dtype=np.float32)
        f = rng.standard_normal(fdims, dtype=np.float32)
        if name == "special":  # signed zeros, infinities, NaN, subnormals
            x.reshape(-1)[:8] = [0.0, -0.0, np.inf, -np.inf, np.nan, 1e-40, -1e-40, 3.0]
        write_wct4(x, HERE / f"{name}_in.wct4")
        write_wct4(f, HERE / f"{name}_flt.wct4")
        base = [sys.executable, "-m", "winconv"]
        subprocess.run(base + ["transform", "--in", str(HERE / f"{name}_in.wct4"), "--layout", "im2win",
                               "--out", str(HERE / f"{name}_win.wct4"), "--hf", str(fdims[2]), "--wf",
                               str(fdims[3]), "--stride", str(stride)], check=True, env=env, stdout=subprocess.DEVNULL)
        subprocess.run(base + ["conv", "--input", str(HERE / f"{name}_in.wct4"), "--filter",
                               str(HERE / f"{name}_flt.wct4"), "--algo", "im2win-opt", "--stride", str(stride),
                               "--out", str(HERE / f"{name}_out.wct4")], check=True, env=env,
                       stdout=subprocess.DEVNULL)
        print(name, "ok")


if __name__ == "__main__":
    main()
