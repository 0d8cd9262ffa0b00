"""Generate golden vectors by running the REFERENCE package (winconv) itself.

Run in the builder container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Outputs (committed, small):
  tests/golden/small_cases.npz   full arrays for Fig. 1, the reference's known-answer
                                 cases and 200 random geometries (the acceptance
                                 generator: pkg/tests/conftest.py:7-31, seed 4242 as in
                                 pkg/tests/test_acceptance.py:128-131), plus special
                                 values (NaN, +-inf, +-0, subnormals)
  tests/golden/layers.json       sha256[:16] checksums of the reference's im2win tensor
                                 and conv output for the 12 benchmark layers at batch 2,
                                 seeds 1000+idx (pkg/tests/test_acceptance.py:57-63), and
                                 config 1 (pad 1 realised as an explicit zero pad)

The GPU box has no /root/reference; tests there regenerate inputs with numpy's
PCG64 (identical bits) and compare against these fixtures.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import winconv as wc  # noqa: E402  (the reference, read-only)
from winconv.kernels.reference import compute_from_windows_basic  # noqa: E402
from winconv.kernels.optimized import compute_from_windows_opt  # noqa: E402

HERE = Path(__file__).resolve().parent


def sha16(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()[:16]


def random_geometry(rng, *, max_filter=7, max_stride=4, max_out=6):
    # pkg/tests/conftest.py:15-31
    h_f = int(rng.integers(1, max_filter + 1))
    w_f = int(rng.integers(1, max_filter + 1))
    stride = int(rng.integers(1, max_stride + 1))
    h_in = h_f + stride * int(rng.integers(0, max_out))
    w_in = w_f + stride * int(rng.integers(0, max_out))
    return dict(batch=int(rng.integers(1, 3)), c_in=int(rng.integers(1, 4)),
                c_out=int(rng.integers(1, 5)), h_f=h_f, w_f=w_f, stride=stride, h_in=h_in, w_in=w_in)


def make_case(rng, *, batch, c_in, c_out, h_f, w_f, stride, h_in, w_in):
    # pkg/tests/conftest.py:7-12
    inp = rng.standard_normal((batch, c_in, h_in, w_in), dtype=np.float32)
    flt = rng.standard_normal((c_out, c_in, h_f, w_f), dtype=np.float32)
    return inp, flt, wc.ConvParams(c_in=c_in, c_out=c_out, h_f=h_f, w_f=w_f, stride=stride)


def record(store: dict, key: str, inp, flt, params):
    t_in = wc.Tensor4(inp)
    windows = wc.im2win(t_in, params)
    direct = wc.conv_direct(t_in, wc.Tensor4(flt), params)
    opt = wc.conv_im2win_opt(t_in, wc.Tensor4(flt), params)
    basic = compute_from_windows_basic(windows, wc.Tensor4(flt), params)
    assert opt == direct and basic == direct, key  # all reference routes agree bitwise
    store[f"{key}/inp"] = inp
    store[f"{key}/flt"] = flt
    store[f"{key}/geom"] = np.array([params.c_in, params.c_out, params.h_f, params.w_f, params.stride])
    store[f"{key}/win"] = windows.data
    store[f"{key}/out"] = opt.data


def main():
    store: dict[str, np.ndarray] = {}
    # Fig. 1 (pkg/tests/test_layouts.py:9-14): 0..26, 2x2 filter, s=1; all-ones filter (test_reference_kernels.py:49-54)
    fig1 = np.arange(27, dtype=np.float32).reshape(1, 3, 3, 3)
    record(store, "fig1", fig1, np.ones((2, 3, 2, 2), np.float32), wc.ConvParams(3, 2, 2, 2, 1))
    # unused edge columns (test_layouts.py:162-170)
    record(store, "edge_cols", np.arange(10, dtype=np.float32).reshape(1, 1, 2, 5),
           np.ones((1, 1, 2, 2), np.float32), wc.ConvParams(1, 1, 2, 2, 2))
    # all-ones 2x2 -> 4 (test_reference_kernels.py:34-40); identity 1x1 (:42-47)
    record(store, "ones", np.ones((1, 1, 3, 3), np.float32), np.ones((1, 1, 2, 2), np.float32),
           wc.ConvParams(1, 1, 2, 2, 1))
    rng = np.random.default_rng(3)
    record(store, "identity1x1", rng.standard_normal((2, 3, 4, 5), dtype=np.float32),
           np.eye(3, dtype=np.float32).reshape(3, 3, 1, 1), wc.ConvParams(3, 3, 1, 1, 1))
    # special values: NaN, +-inf, +-0, subnormals flow through bit-exactly
    sp = rng.standard_normal((2, 2, 6, 7), dtype=np.float32)
    sp[0, 0, 0, 0] = np.nan
    sp[0, 1, 2, 3] = np.inf
    sp[1, 0, 4, 4] = -np.inf
    sp[1, 1, 1, 1] = -0.0
    sp[1, 1, 5, 6] = np.float32(1e-40)
    fsp = rng.standard_normal((3, 2, 3, 2), dtype=np.float32)
    fsp[2, 1, 0, 0] = -0.0
    t_in, t_f, p = wc.Tensor4(sp), wc.Tensor4(fsp), wc.ConvParams(2, 3, 3, 2, 1)
    store["special/inp"], store["special/flt"] = sp, fsp
    store["special/geom"] = np.array([2, 3, 3, 2, 1])
    store["special/win"] = wc.im2win(t_in, p).data
    store["special/out"] = wc.conv_im2win_opt(t_in, t_f, p).data
    # 200 random geometries (acceptance generator, seed 4242)
    rng = np.random.default_rng(4242)
    for i in range(200):
        inp, flt, params = make_case(rng, **random_geometry(rng))
        record(store, f"rand{i:03d}", inp, flt, params)
    np.savez_compressed(HERE / "small_cases.npz", **store)

    layers = {}
    for idx, (name, cfg) in enumerate(wc.BENCHMARKS.items()):
        cfg = replace(cfg, batch=2, seed=1000 + idx)
        inp, flt = wc.bench.make_inputs(cfg)
        windows = wc.im2win(inp, cfg.params)
        out = compute_from_windows_opt(windows, flt, cfg.params)
        layers[name] = dict(batch=2, seed=1000 + idx, win_sha=sha16(windows.data),
                            out_sha=sha16(out.data), out_abs_sum=float(np.abs(out.data.astype(np.float64)).sum()))
        print(name, layers[name], flush=True)
    # config 1: N=8 C=64 56x56 K=64 3x3 s1 pad1 -> explicit zero pad to 58x58
    rng = np.random.default_rng(0)
    x = rng.standard_normal((8, 64, 56, 56), dtype=np.float32)
    f = rng.standard_normal((64, 64, 3, 3), dtype=np.float32)
    xp = np.zeros((8, 64, 58, 58), np.float32)
    xp[:, :, 1:57, 1:57] = x
    params = wc.ConvParams(64, 64, 3, 3, 1)
    out = wc.conv_im2win_opt(wc.Tensor4(xp), wc.Tensor4(f), params)
    layers["cfg1-pad1"] = dict(batch=8, seed=0, draw="56x56 then zero-pad", out_sha=sha16(out.data),
                               win_sha=sha16(wc.im2win(wc.Tensor4(xp), params).data))
    # the survey's checksum for config 1 drew the operands at the padded size via make_inputs
    cfg1 = wc.BenchConfig(name="cfg1", c_in=64, h_in=58, w_in=58, c_out=64, h_f=3, w_f=3, stride=1, batch=8, seed=0)
    inp, flt = wc.bench.make_inputs(cfg1)
    out = wc.conv_im2win_opt(inp, flt, params)
    layers["cfg1-58x58"] = dict(batch=8, seed=0, draw="make_inputs at 58x58", out_sha=sha16(out.data))
    print(layers["cfg1-pad1"], layers["cfg1-58x58"])
    (HERE / "layers.json").write_text(json.dumps(layers, indent=1) + "\n")


if __name__ == "__main__":
    main()
