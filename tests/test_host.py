"""Host-side logic (no GPU): geometry, plans, errors, footprints, fixtures, the C-ABI library."""

import re
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2306_14316_b200 as pkg
from paper_2306_14316_b200 import _lib
from paper_2306_14316_b200.plan import simt_tile_for, to_c_plan

ROOT = Path(__file__).resolve().parent.parent

# pkg/tests/test_acceptance.py:24-37 (paper Table 2)
TABLE2_OUTPUTS = {
    "conv1": (96, 55, 55), "conv2": (96, 56, 56), "conv3": (64, 111, 111), "conv4": (64, 109, 109),
    "conv5": (256, 20, 20), "conv6": (512, 10, 10), "conv7": (64, 222, 222), "conv8": (128, 110, 110),
    "conv9": (64, 54, 54), "conv10": (128, 26, 26), "conv11": (256, 12, 12), "conv12": (512, 5, 5),
}


def test_table2_geometry():
    for name, cfg in pkg.BENCHMARKS.items():
        assert (cfg.c_out, *cfg.out_dims) == TABLE2_OUTPUTS[name], name


def test_flops_formula():
    cfg = pkg.BENCHMARKS["conv1"]
    assert cfg.flops == 2 * 2 * 96 * 55 * 55 * 3 * 11 * 11


def test_conv_params_validation():
    with pytest.raises(pkg.GeometryError):
        pkg.ConvParams(0, 1, 3, 3, 1)
    with pytest.raises(pkg.GeometryError):
        pkg.ConvParams(1, 1, 3, 3, 0)
    with pytest.raises(pkg.GeometryError):
        pkg.output_dims(2, 5, pkg.ConvParams(1, 1, 3, 3, 1))
    assert pkg.output_dims(224, 224, pkg.ConvParams(64, 64, 7, 7, 2)) == (109, 109)
    assert pkg.effective_width(109, 7, 2) == 223


def test_tile_plan_validation():
    with pytest.raises(pkg.PlanError):
        pkg.TilePlan(m_b=6, n_b=8, k_b=4, m_t=4, n_t=2)
    with pytest.raises(pkg.PlanError):
        pkg.TilePlan(m_b=0, n_b=8, k_b=4, m_t=1, n_t=2)
    plan = pkg.TilePlan(m_b=8, n_b=8, k_b=4, m_t=4, n_t=4, micro_kernel=False)
    assert (plan.m_t, plan.n_t) == (1, 1) and plan.workers_per_block == 64
    for cfg in pkg.BENCHMARKS.values():
        p = pkg.default_plan(cfg.gemm_dims())
        assert p.m_b % p.m_t == 0 and p.n_b % p.n_t == 0
    assert pkg.default_plan(pkg.GemmDims(1, 500, 64)).m_b == 1


def test_plan_to_c_abi():
    assert to_c_plan(None) is None
    c = to_c_plan(pkg.TilePlan(64, 256, 16, 8, 8))
    assert (c.block_cfg, c.micro_kernel, c.vectorized_load, c.prefetch_double_buffer) == (1, 1, 1, 1)
    c = to_c_plan(pkg.TilePlan(64, 128, 128, 8, 8, prefetch_double_buffer=False, vectorized_load=False))
    assert (c.block_cfg, c.vectorized_load, c.prefetch_double_buffer) == (-1, 0, 0)
    c = to_c_plan(pkg.TilePlan(64, 128, 128, 8, 8, micro_kernel=False))
    assert c.micro_kernel == 0
    assert pkg.gpu_plan(pkg.BENCHMARKS["conv4"].gemm_dims()).m_b == 64
    assert simt_tile_for(pkg.GemmDims(96, 10 ** 6, 363)) == 2


def test_gemm_index_roundtrip():
    for n in range(0, 2 * 5 * 7):
        assert pkg.compose_n(*pkg.decompose_n(n, 5, 7), 5, 7) == n
    for k in range(0, 3 * 4 * 5):
        assert pkg.compose_k(*pkg.decompose_k(k, 4, 5), 4, 5) == k


def test_footprints_match_reference_counts():
    p = pkg.ConvParams(3, 96, 11, 11, 4)
    assert pkg.footprint_elems("im2col", 1, 3, 227, 227, p) == 1_098_075
    assert pkg.footprint_elems("im2win", 1, 3, 227, 227, p) == 412_005
    assert pkg.footprint_elems("raw", 1, 3, 227, 227, p) == 154_587
    f1 = pkg.ConvParams(3, 2, 2, 2, 1)
    assert [pkg.footprint_elems(l, 1, 3, 3, 3, f1) for l in ("raw", "im2col", "im2win")] == [27, 48, 36]
    with pytest.raises(ValueError):
        pkg.footprint_elems("nchw", 1, 3, 3, 3, f1)


def test_max_rel_diff_semantics():
    a = np.array([[[[1.0, -0.0, np.nan, 10.0]]]], np.float32)
    b = np.array([[[[1.0, 0.0, np.nan, 11.0]]]], np.float32)
    assert pkg.max_rel_diff(a, a) == 0.0
    assert pkg.max_rel_diff(a[..., :2], b[..., :2]) == 0.0   # |diff|=0 for +-0
    assert abs(pkg.max_rel_diff(a[..., 3:], b[..., 3:]) - 1 / 11) < 1e-12
    with pytest.raises(pkg.ShapeError):
        pkg.max_rel_diff(a, b[..., :2])


def test_fixture_roundtrip(tmp_path):
    x = np.random.default_rng(0).standard_normal((1, 2, 3, 4)).astype(np.float32)
    x[0, 0, 0, 0] = np.nan
    x[0, 0, 0, 1] = -0.0
    pkg.write_tensor(x, tmp_path / "a.wct4")
    y = pkg.read_tensor(tmp_path / "a.wct4")
    assert (x.view(np.uint32) == y.view(np.uint32)).all()
    (tmp_path / "bad").write_bytes(b"XXXX" + bytes(40))
    with pytest.raises(pkg.FixtureFormatError):
        pkg.read_tensor(tmp_path / "bad")


def test_c_abi_library_exports_every_header_symbol():
    header = (ROOT / "include" / "im2win_sm100.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|size_t|const char\*|int32_t|int64_t)\s+(im2win_\w+)\s*\(", header, re.M))
    assert declared == set(_lib.EXPORTED_SYMBOLS)
    lib = _lib.load()
    for sym in declared:
        assert hasattr(lib, sym), sym
    assert lib.im2win_abi_version() == 100
    assert lib.im2win_conv_workspace_bytes(64, 64, 3, 3, 0) > 64 * 64 * 9 * 4


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    with pytest.raises(pkg.ShapeError, match="CUDA"):
        pkg.Tensor4(np.zeros((1, 1, 4, 4), np.float32))


def test_tile_pick_mirrors_library():
    """plan.simt_tile_for restates im2win_simt_pick (csrc/conv_simt.cu); no GPU call involved."""
    import ctypes

    from paper_2306_14316_b200 import _lib

    lib = _lib.load()
    lib.im2win_simt_pick.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_int]
    lib.im2win_simt_pick.restype = ctypes.c_int
    for batch in (1, 2, 8, 32, 128, 256):
        for name, cfg in pkg.BENCHMARKS.items():
            d = cfg.gemm_dims()
            d = pkg.GemmDims(d.m, d.n // cfg.batch * batch, d.k)
            assert simt_tile_for(d) == lib.im2win_simt_pick(d.m, d.n, d.k), (name, batch)
    for m in (1, 32, 64, 96, 100, 192, 512):
        for n in (1, 1000, 10 ** 5, 3 * 10 ** 6):
            assert simt_tile_for(pkg.GemmDims(m, n, 9)) == lib.im2win_simt_pick(m, n, 9), (m, n)


def test_output_dims_with_padding():
    p = pkg.ConvParams(64, 64, 3, 3, 1, pad=1)
    assert pkg.output_dims(56, 56, p) == (56, 56)
    assert pkg.output_dims(224, 224, pkg.ConvParams(3, 64, 7, 7, 2, pad=3)) == (112, 112)
    assert pkg.output_dims(2, 2, pkg.ConvParams(1, 1, 3, 3, 1, pad=1)) == (2, 2)
    with pytest.raises(pkg.GeometryError):
        pkg.ConvParams(1, 1, 3, 3, 1, pad=-1)
    with pytest.raises(pkg.GeometryError):
        pkg.output_dims(1, 1, pkg.ConvParams(1, 1, 5, 5, 1, pad=1))
    assert pkg.ConvParams(1, 1, 3, 3) == pkg.ConvParams(1, 1, 3, 3, 1, 0)


def test_footprint_report_dominance():
    """Reference acceptance criterion: the window layout is smaller than im2col on every layer
    (test_acceptance.py:84-103); the report carries the same counts as footprint_elems."""
    from dataclasses import replace

    rows = pkg.footprint_report([replace(c, batch=1) for c in pkg.BENCHMARKS.values()])
    assert [r.name for r in rows] == list(pkg.BENCHMARKS)
    for r, cfg in zip(rows, pkg.BENCHMARKS.values()):
        assert r.raw_elems < r.im2win_elems < r.im2col_elems
        assert r.im2win_elems == pkg.footprint_elems("im2win", 1, cfg.c_in, cfg.h_in, cfg.w_in, cfg.params)
        assert 0 < r.reduction_pct < 100
    assert rows[0].im2win_elems == 412_005


def test_harness_names_match_reference():
    assert pkg.ALGORITHMS[0] == "im2win-opt" and "cudnn" in pkg.ALGORITHMS
    from paper_2306_14316_b200 import harness

    assert harness.ABLATION_VARIANTS == ("full", "-prefetch-double-buffer", "-vectorized-load", "-micro-kernel")
    assert harness.CSV_COLUMNS[:17] == ("name", "algorithm", "variant", "batch", "repeats", "h_o", "w_o", "flops",
                                        "transform_s", "compute_s", "total_s", "tflops", "raw_elems",
                                        "im2col_elems", "im2win_elems", "footprint_reduction_pct", "checksum")


def test_bench_config_is_the_reference_dataclass():
    """BenchConfig carries the reference's fields and defaults (bench.py:43-59), so
    replace(BENCHMARKS[n], batch=N, repeats=R, algorithm=...) works unchanged."""
    import dataclasses
    import inspect

    from paper_2306_14316_b200 import harness
    from paper_2306_14316_b200.workloads import BENCHMARKS, BenchConfig

    fields = [(f.name, f.default) for f in dataclasses.fields(BenchConfig)]
    assert [n for n, _ in fields] == ["name", "c_in", "h_in", "w_in", "c_out", "h_f", "w_f", "stride", "batch",
                                      "repeats", "algorithm", "plan", "seed"]
    assert dict(fields)["repeats"] == 10 and dict(fields)["algorithm"] == "im2win-opt"
    assert dict(fields)["plan"] is None and dict(fields)["batch"] == 2 and dict(fields)["seed"] == 0
    cfg = dataclasses.replace(BENCHMARKS["conv9"], batch=8, repeats=3, algorithm="im2win-opt")
    assert (cfg.batch, cfg.repeats, cfg.algorithm) == (8, 3, "im2win-opt")
    sig = inspect.signature(harness.run_bench)
    assert list(sig.parameters)[:2] == ["cfg", "variant"] and sig.parameters["variant"].default == "-"
    assert sig.parameters["device"].kind is inspect.Parameter.KEYWORD_ONLY
    assert list(inspect.signature(harness.search_plan).parameters)[:3] == ["cfg", "grid", "repeats"]
    # the reference's CPU baselines resolve to their GPU counterparts
    assert set(harness.REFERENCE_ALIASES) == {"direct", "im2col-gemm", "implicit-gemm"}
    assert all(a in harness.ALGORITHMS for a in harness.REFERENCE_ALIASES.values())
