"""GPU parity: the sm_100a kernels vs the reference's goldens and the CPU oracle.

Bar (BASELINE.json north_star): im2win transform bit-exact; FP32 conv within
1e-5 -> achieved as bitwise equality (fp32-exact variant); fp32-fma within 1e-4.
All calls go through the package's public API, which calls the C ABI.
"""

from dataclasses import replace

import numpy as np
import pytest
import torch

from conftest import bits_equal, bits_equal_nan_as_class
from oracle import oracle as orc
import paper_2306_14316_b200 as pkg
from paper_2306_14316_b200.workloads import BENCHMARKS, make_config1_inputs, make_inputs

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _params(c):
    return pkg.ConvParams(c["c_in"], c["c_out"], c["h_f"], c["w_f"], c["stride"])


def test_library_is_native():
    from paper_2306_14316_b200 import _lib
    assert _lib.load().im2win_abi_version() == 100
    assert torch.cuda.get_device_capability(0) == (10, 0)


def test_transform_bit_exact_small_cases(small_cases):
    for name, c in small_cases.items():
        w = pkg.im2win(torch.from_numpy(c["inp"]).to(DEV), _params(c))
        assert bits_equal(w.data.cpu().numpy(), c["win"]), name


def test_conv_bit_exact_small_cases(small_cases):
    for name, c in small_cases.items():
        out = pkg.conv_im2win_opt(torch.from_numpy(c["inp"]).to(DEV), torch.from_numpy(c["flt"]).to(DEV), _params(c))
        assert bits_equal_nan_as_class(out.numpy(), c["out"]), name


@pytest.mark.parametrize("variant", ["fp32-fma"])
def test_conv_fma_within_1e4(small_cases, variant):
    for name, c in list(small_cases.items())[:80]:
        if name == "special":
            continue
        out = pkg.conv_im2win_opt(torch.from_numpy(c["inp"]).to(DEV), torch.from_numpy(c["flt"]).to(DEV),
                                  _params(c), variant=variant)
        assert pkg.max_rel_diff(out, c["out"]) <= 1e-4, name


def test_all_tiles_and_toggles_bitwise(small_cases):
    names = ["fig1", "special", "identity1x1"] + [f"rand{i:03d}" for i in range(0, 200, 7)]
    for name in names:
        c = small_cases[name]
        inp = torch.from_numpy(c["inp"]).to(DEV)
        flt = torch.from_numpy(c["flt"]).to(DEV)
        w = pkg.im2win(inp, _params(c))
        for (bm, bn) in pkg.plan.SIMT_TILES:
            for mk in (True, False):
                for vec in (True, False):
                    for pf in (True, False):
                        plan = pkg.TilePlan(bm, bn, 8, 8, 8, micro_kernel=mk, vectorized_load=vec,
                                            prefetch_double_buffer=pf)
                        out = pkg.compute_from_windows_opt(w, flt, _params(c), plan)
                        assert bits_equal_nan_as_class(out.numpy(), c["out"]), (name, plan)
        for (bm, bn) in pkg.plan.SIMT_TILES_MT4:
            plan = pkg.TilePlan(bm, bn, 8, 4, 4)
            out = pkg.compute_from_windows_opt(w, flt, _params(c), plan)
            assert bits_equal_nan_as_class(out.numpy(), c["out"]), (name, plan)


@pytest.mark.parametrize("name", list(BENCHMARKS))
def test_layer_checksums_bitwise(name, layer_goldens):
    g = layer_goldens[name]
    cfg = replace(BENCHMARKS[name], batch=g["batch"], seed=g["seed"])
    inp, flt = make_inputs(cfg)
    w = pkg.im2win(torch.from_numpy(inp).to(DEV), cfg.params)
    assert orc.checksum(w.data.cpu().numpy()) == g["win_sha"]
    out = pkg.compute_from_windows_opt(w, torch.from_numpy(flt).to(DEV), cfg.params)
    assert orc.checksum(out.numpy()) == g["out_sha"]
    # every compiled CTA tile gives the same bits
    for (bm, bn) in pkg.plan.SIMT_TILES:
        o2 = pkg.compute_from_windows_opt(w, torch.from_numpy(flt).to(DEV), cfg.params,
                                          pkg.TilePlan(bm, bn, 8, 8, 8))
        assert o2 == out, (name, bm, bn)
    for (bm, bn) in pkg.plan.SIMT_TILES_MT4:
        o2 = pkg.compute_from_windows_opt(w, torch.from_numpy(flt).to(DEV), cfg.params,
                                          pkg.TilePlan(bm, bn, 8, 4, 4))
        assert o2 == out, (name, bm, bn, "mt4")


def test_config1_checksum(layer_goldens):
    inp, flt = make_config1_inputs(0)
    out = pkg.conv_im2win_opt(inp, flt, pkg.ConvParams(64, 64, 3, 3, 1))
    assert orc.checksum(out.numpy()) == layer_goldens["cfg1-pad1"]["out_sha"]


@pytest.mark.parametrize("name,batch", [("conv1", 128), ("conv7", 128), ("conv9", 128), ("conv12", 128),
                                        ("conv4", 64), ("conv5", 128), ("conv6", 128), ("conv10", 128)])
def test_large_batch_sampled_images(name, batch):
    """Full-size runs: images are independent (reference.py:78-90), so sampled
    images checked against the oracle give the bits of the whole batch.  conv5/conv10
    and conv6 at N=128 take the SIMT tail split (the last images come from the 4x4-tile launch)."""
    cfg = replace(BENCHMARKS[name], batch=batch, seed=7)
    g = torch.Generator(device="cpu").manual_seed(7)
    inp = torch.randn((batch, cfg.c_in, cfg.h_in, cfg.w_in), generator=g)
    flt = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), generator=g)
    out = pkg.conv_im2win_opt(inp.to(DEV), flt.to(DEV), cfg.params)
    win = pkg.im2win(inp.to(DEV), cfg.params)
    for i in (0, batch // 2 + 1, batch - 1):
        ref = orc.conv_direct(inp[i:i + 1].numpy(), flt.numpy(), cfg.stride)
        assert bits_equal(out.data[i:i + 1].cpu().numpy(), ref), (name, i)
        refw = orc.im2win_fill(inp[i:i + 1].numpy(), cfg.h_f, cfg.w_f, cfg.stride)
        assert bits_equal(win.data[i:i + 1].cpu().numpy(), refw), (name, i)


def test_deterministic_and_stream_safe():
    cfg = replace(BENCHMARKS["conv10"], batch=16, seed=3)
    inp, flt = make_inputs(cfg)
    a = pkg.conv_im2win_opt(inp, flt, cfg.params)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        b = pkg.conv_im2win_opt(inp, flt, cfg.params)
    s.synchronize()
    assert a == b


def test_errors_raise_before_launch():
    x = torch.randn(1, 3, 8, 8, device=DEV)
    with pytest.raises(pkg.ShapeError):
        pkg.im2win(x, pkg.ConvParams(4, 1, 3, 3, 1))
    with pytest.raises(pkg.GeometryError):
        pkg.im2win(x, pkg.ConvParams(3, 1, 9, 3, 1))
    with pytest.raises(pkg.ShapeError):
        pkg.conv_im2win_opt(x, torch.randn(2, 3, 3, 3, device=DEV), pkg.ConvParams(3, 1, 3, 3, 1))


# ---------------------------------------------------------------- tensor-core variants
# Stated tolerances: normalized max|d|/rms(ref)
# TF32 <= 1e-2, BF16 <= 4e-2 (operands rounded to nearest, fp32 accumulation).
TC_TOL = {"tf32": 1e-2, "bf16": 4e-2}


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
@pytest.mark.parametrize("name", list(BENCHMARKS))
def test_tc_layers_within_tolerance(name, variant, layer_goldens):
    g = layer_goldens[name]
    cfg = replace(BENCHMARKS[name], batch=g["batch"], seed=g["seed"])
    inp, flt = make_inputs(cfg)
    out = pkg.conv_im2win_opt(inp, flt, cfg.params, variant=variant).numpy()
    ref = orc.conv_direct(inp, flt, cfg.stride)
    assert orc.checksum(ref) == g["out_sha"]
    assert pkg.normalized_max_diff(out, ref) <= TC_TOL[variant], name


# Element-wise error bound of a tensor-core result: operands rounded to tf32 (10 stored
# mantissa bits, truncated in hardware: u = 2^-10 per operand) or bf16 (8 significant bits, RN: u = 2^-8), fp32
# accumulation over K terms.  |out - ref| <= (2u + u^2 + (K + 2) 2^-24) * conv(|x|, |w|).
TC_UNIT = {"tf32": 2.0 ** -10, "bf16": 2.0 ** -8}


def _tc_elementwise_ok(out, ref, inp, flt, stride, variant):
    """Finite reference entries within the rounding bound; NaN and +-inf reproduced as classes."""
    u = TC_UNIT[variant]
    k = flt.shape[1] * flt.shape[2] * flt.shape[3]
    a = orc.conv_direct(np.abs(inp), np.abs(flt), stride).astype(np.float64)
    fin = np.isfinite(ref)
    bound = (2 * u + u * u + (k + 2) * 2.0 ** -24) * a * 1.001
    with np.errstate(invalid="ignore"):
        err = np.abs(out.astype(np.float64) - ref.astype(np.float64))
    ok_fin = bool((err[fin] <= bound[fin]).all())
    ok_nan = bool((np.isnan(out) == np.isnan(ref)).all())
    inf = np.isinf(ref)
    ok_inf = bool((out[inf] == ref[inf]).all())
    return ok_fin and ok_nan and ok_inf


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
def test_tc_small_cases(small_cases, variant):
    """Every reference small case (Fig. 1, the pkg/tests known answers, 200 random geometries,
    and the NaN/+-inf/-0/subnormal case): within the stated normalized tolerance and within
    the element-wise rounding bound; NaN and +-inf outputs where the reference has them."""
    for name, c in small_cases.items():
        params = _params(c)
        out = pkg.conv_im2win_opt(torch.from_numpy(c["inp"]).to(DEV), torch.from_numpy(c["flt"]).to(DEV),
                                  params, variant=variant).numpy()
        ref = c["out"]
        assert _tc_elementwise_ok(out, ref, c["inp"], c["flt"], params.stride, variant), name
        if name != "special":  # the normalized metric needs a finite reference
            assert pkg.normalized_max_diff(out, ref) <= TC_TOL[variant], name


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
def test_tc_special_values(variant):
    """TC behaviour on special inputs, stated: NaN in a window -> NaN output; +-inf -> +-inf
    (inf * 0 -> NaN, as in IEEE); -0 and subnormal inputs act as (+-)0 within the bound."""
    rng = np.random.default_rng(5)
    inp = rng.standard_normal((2, 8, 9, 9), dtype=np.float32)
    flt = rng.standard_normal((16, 8, 3, 3), dtype=np.float32)
    inp[0, 0, 0, 0] = np.nan
    inp[0, 3, 4, 4] = np.inf
    inp[1, 5, 8, 8] = -np.inf
    inp[1, 2, 2, 2] = -0.0
    inp[1, 6, 3, 3] = np.float32(1e-40)
    flt[3, 3, 1, 1] = 0.0  # inf * 0 -> NaN for output channel 3
    params = pkg.ConvParams(8, 16, 3, 3, 1)
    ref = orc.conv_direct(inp, flt, 1)
    for tc_path in ("auto", "fused", "gather"):
        out = pkg.conv_im2win_opt(inp, flt, params, variant=variant, tc_path=tc_path).numpy()
        assert np.isnan(out[0, :, 0, 0]).all() and np.isnan(out[0, 3, 3, 3]), tc_path  # NaN; inf * 0
        assert np.isinf(out[0, 3, 2:5, 2:5]).sum() == 8, tc_path  # the other taps over the inf: +-inf
        assert _tc_elementwise_ok(out, ref, inp, flt, 1, variant), tc_path


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
def test_tc_large_batch_sampled_images(variant):
    cfg = replace(BENCHMARKS["conv8"], batch=128, seed=11)
    g = torch.Generator(device="cpu").manual_seed(11)
    inp = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), generator=g)
    flt = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), generator=g)
    out = pkg.conv_im2win_opt(inp.to(DEV), flt.to(DEV), cfg.params, variant=variant)
    for i in (0, 77, 127):
        ref = orc.conv_direct(inp[i:i + 1].numpy(), flt.numpy(), cfg.stride)
        assert pkg.normalized_max_diff(out.data[i:i + 1].cpu().numpy(), ref) <= TC_TOL[variant]


@pytest.mark.parametrize("tc_path", ["fused", "cl", "gather"])
@pytest.mark.parametrize("variant", ["tf32", "bf16"])
def test_tc_paths_all_layers(tc_path, variant, layer_goldens):
    """Every tensor-core path (fused TMA windows / materialised channels-last Ĩ /
    gathered reference Ĩ) stays within the stated tolerance on the 12 layers."""
    for name in BENCHMARKS:
        g = layer_goldens[name]
        cfg = replace(BENCHMARKS[name], batch=g["batch"], seed=g["seed"])
        inp, flt = make_inputs(cfg)
        ref = orc.conv_direct(inp, flt, cfg.stride)
        out = pkg.conv_im2win_opt(inp, flt, cfg.params, variant=variant, tc_path=tc_path).numpy()
        assert pkg.normalized_max_diff(out, ref) <= TC_TOL[variant], (name, tc_path)


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
def test_tc_fused_odd_geometries(variant):
    """Fused path edge cases: partial pixel tiles, strides, Co not a multiple of the
    UMMA N tile, multi-image boxes, tiny images."""
    rng = np.random.default_rng(21)
    cases = [(3, 16, 9, 11, 20, 3, 3, 1), (2, 32, 13, 13, 40, 5, 3, 2), (5, 64, 7, 7, 130, 3, 3, 1),
             (1, 8, 4, 4, 3, 2, 2, 1), (4, 96, 10, 9, 257, 1, 1, 1), (2, 16, 33, 31, 17, 7, 5, 3)]
    for (n, c, h, w, co, hf, wf, s) in cases:
        inp = rng.standard_normal((n, c, h, w), dtype=np.float32)
        flt = rng.standard_normal((co, c, hf, wf), dtype=np.float32)
        params = pkg.ConvParams(c, co, hf, wf, s)
        ref = orc.conv_direct(inp, flt, s)
        out = pkg.conv_im2win_opt(inp, flt, params, variant=variant, tc_path="fused").numpy()
        assert pkg.normalized_max_diff(out, ref) <= TC_TOL[variant], (n, c, h, w, co, hf, wf, s)


def test_basic_kernel_bitwise(small_cases):
    """Paper Alg. 2 basic kernel (reference compute_from_windows_basic) is bit-exact too."""
    for name in ["fig1", "special", "identity1x1"] + [f"rand{i:03d}" for i in range(0, 200, 3)]:
        c = small_cases[name]
        out = pkg.conv_im2win_basic(torch.from_numpy(c["inp"]).to(DEV), torch.from_numpy(c["flt"]).to(DEV), _params(c))
        assert bits_equal_nan_as_class(out.numpy(), c["out"]), name


def test_harness_records_and_csv():
    from paper_2306_14316_b200 import harness
    cfg = replace(BENCHMARKS["conv10"], batch=4, seed=5)
    recs = [harness.run_bench(replace(cfg, repeats=2, algorithm=a))
            for a in ("im2win-opt", "im2win-basic", "im2win-bf16", "cudnn")]
    assert recs[0].checksum == recs[1].checksum          # exact kernels agree bitwise
    assert all(r.tflops > 0 and r.total_s > 0 for r in recs)
    abl = harness.run_ablation(replace(cfg, repeats=2))
    assert [r.variant for r in abl] == list(harness.ABLATION_VARIANTS)
    assert len({r.checksum for r in abl}) == 1 and abl[0].checksum == recs[0].checksum
    csv = harness.report_csv(recs + abl)
    assert csv.splitlines()[0].split(",")[:17] == list(harness.CSV_COLUMNS[:17])


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
def test_tc_fused_padded_channels(variant):
    """C not a multiple of 16 bytes (C=3 layers conv1/2/3/7, C=5, C=6): the channels-last
    copy pads the channel pitch with zeros and the fused/shift kernels still apply."""
    rng = np.random.default_rng(33)
    for (n, c, h, w, co, hf, wf, s) in [(2, 3, 227, 227, 96, 11, 11, 4), (2, 3, 40, 44, 64, 3, 3, 1),
                                        (3, 5, 17, 19, 20, 5, 5, 1), (2, 6, 21, 20, 33, 7, 7, 2)]:
        inp = rng.standard_normal((n, c, h, w), dtype=np.float32)
        flt = rng.standard_normal((co, c, hf, wf), dtype=np.float32)
        params = pkg.ConvParams(c, co, hf, wf, s)
        ref = orc.conv_direct(inp, flt, s)
        out = pkg.conv_im2win_opt(inp, flt, params, variant=variant).numpy()
        assert pkg.normalized_max_diff(out, ref) <= TC_TOL[variant], (c, hf, s)


@pytest.mark.slow
def test_64bit_indexing_conv4_n256():
    """at N=256, conv4's Ĩ has 2.79e9 > 2^31 elements.  Sampled images at the
    far end of the batch must still be bit-exact (64-bit offsets in transform and conv)."""
    cfg = replace(BENCHMARKS["conv4"], batch=256, seed=13)
    g = torch.Generator(device="cpu").manual_seed(13)
    flt = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), generator=g)
    x = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), generator=g)
    win = pkg.im2win(x.to(DEV), cfg.params)
    assert win.elements() > 2 ** 31
    out = pkg.compute_from_windows_opt(win, flt.to(DEV), cfg.params)
    for i in (0, 200, 255):
        ref_w = orc.im2win_fill(x[i:i + 1].numpy(), cfg.h_f, cfg.w_f, cfg.stride)
        assert bits_equal(win.data[i:i + 1].cpu().numpy(), ref_w), i
        ref = orc.conv_direct(x[i:i + 1].numpy(), flt.numpy(), cfg.stride)
        assert bits_equal(out.data[i:i + 1].cpu().numpy(), ref), i


@pytest.mark.parametrize("name", ["conv1", "conv4", "conv9", "conv12"])
def test_host_pipeline_matches_goldens(name, layer_goldens):
    """conv_im2win_opt_host (numpy in -> host out, streamed chunks) gives the reference's bits."""
    g = layer_goldens[name]
    cfg = replace(BENCHMARKS[name], batch=g["batch"], seed=g["seed"])
    inp, flt = make_inputs(cfg)
    for chunk in (0, 1):
        out = pkg.conv_im2win_opt_host(inp, flt, cfg.params, chunk_images=chunk)
        assert not out.is_cuda
        assert orc.checksum(out.numpy()) == g["out_sha"], (name, chunk)


@pytest.mark.parametrize("variant", pkg.VARIANTS)
def test_host_pipeline_equals_device_path(variant):
    """Every chunking of the streamed host path is bit-identical to the device path (ragged last chunk)."""
    cfg = replace(BENCHMARKS["conv10"], batch=11, seed=5)
    inp, flt = make_inputs(cfg)
    if variant in ("tf32", "bf16"):
        dev = pkg.conv_im2win_opt(inp, flt, cfg.params, variant=variant).numpy()
    else:
        dev = pkg.conv_im2win_opt(inp, flt, cfg.params, variant=variant).numpy()
    pinned_in = torch.from_numpy(inp).pin_memory()
    out = torch.empty(dev.shape, dtype=torch.float32).pin_memory()
    for chunk in (0, 1, 4, 11, 64):
        out.fill_(float("nan"))
        pkg.conv_im2win_opt_host(pinned_in, flt, cfg.params, variant=variant, chunk_images=chunk, out=out)
        assert bits_equal(out.numpy(), dev), (variant, chunk)


def test_host_pipeline_errors():
    cfg = replace(BENCHMARKS["conv12"], batch=2, seed=1)
    inp, flt = make_inputs(cfg)
    with pytest.raises(pkg.ShapeError):
        pkg.conv_im2win_opt_host(inp[:, :5], flt, cfg.params)
    with pytest.raises(pkg.ShapeError):
        pkg.conv_im2win_opt_host(torch.from_numpy(inp).to(DEV), flt, cfg.params)
    with pytest.raises(pkg.GeometryError):
        pkg.conv_im2win_opt_host(inp[:, :, :2, :2], flt, cfg.params)
    with pytest.raises(pkg.ShapeError):
        pkg.conv_im2win_opt_host(inp, flt, cfg.params, out=torch.empty(3))


def test_host_pipeline_nonblocking_overlapped_submissions():
    """Several non-blocking submissions in flight at once give the blocking path's bits."""
    names = ["conv9", "conv10", "conv12", "conv9"]
    jobs = []
    for i, name in enumerate(names):
        cfg = replace(BENCHMARKS[name], batch=7 + i, seed=40 + i)
        inp, flt = make_inputs(cfg)
        ref = pkg.conv_im2win_opt_host(inp, flt, cfg.params).clone()
        h = pkg.conv_im2win_opt_host(torch.from_numpy(inp).pin_memory(), flt, cfg.params, chunk_images=2,
                                     wait=False)
        jobs.append((h, ref))
    for h, ref in reversed(jobs):
        assert bits_equal(h.wait().numpy(), ref.numpy())


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
@pytest.mark.parametrize("select", ["phase", "shift", "generic"])
def test_tc_kernel_selections_all_layers(select, variant, layer_goldens, monkeypatch):
    """Each fused tensor-core kernel (phase-shift / window-shift / generic TMA window) is
    within tolerance on every layer where it applies (forced through the library's env switches)."""
    env = {"phase": ("2", "0"), "shift": ("0", "2"), "generic": ("0", "0")}[select]
    monkeypatch.setenv("IM2WIN_PHASE", env[0])
    monkeypatch.setenv("IM2WIN_SHIFT", env[1])
    for name in BENCHMARKS:
        g = layer_goldens[name]
        cfg = replace(BENCHMARKS[name], batch=g["batch"], seed=g["seed"])
        inp, flt = make_inputs(cfg)
        ref = orc.conv_direct(inp, flt, cfg.stride)
        out = pkg.conv_im2win_opt(inp, flt, cfg.params, variant=variant, tc_path="fused").numpy()
        assert pkg.normalized_max_diff(out, ref) <= TC_TOL[variant], (name, select)


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
def test_tc_phase_kernel_edge_geometries(variant, monkeypatch):
    """Phase kernel on ragged geometries: odd/even H and W, stride 2 and 1, Wf 3/5/7, multi-row
    tiles, an odd number of pixel tiles (the second tile of the last pair is empty)."""
    monkeypatch.setenv("IM2WIN_PHASE", "2")
    cases = [(3, 64, 17, 19, 64, 7, 7, 2), (2, 32, 30, 31, 96, 5, 5, 2), (1, 64, 23, 9, 64, 3, 3, 2),
             (2, 40, 12, 13, 128, 3, 3, 1), (1, 64, 140, 140, 64, 7, 7, 2), (5, 32, 8, 8, 64, 5, 5, 1)]
    for (n, c, h, w, co, hf, wf, s) in cases:
        rng = np.random.default_rng(n * 1000 + h)
        inp = rng.standard_normal((n, c, h, w), dtype=np.float32)
        flt = rng.standard_normal((co, c, hf, wf), dtype=np.float32)
        ref = orc.conv_direct(inp, flt, s)
        out = pkg.conv_im2win_opt(inp, flt, pkg.ConvParams(c, co, hf, wf, s), variant=variant,
                                  tc_path="fused").numpy()
        assert pkg.normalized_max_diff(out, ref) <= TC_TOL[variant], (n, c, h, w, co, hf, wf, s)


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
def test_tc_phase_tap_pairs(variant, monkeypatch, layer_goldens):
    """Tap pairs per MMA (IM2WIN_PHASE_TN2=2; B rows 64-127 = the next tap, D[p] + D[p+1] shifted
    in the epilogue, odd last taps as N=64 MMAs): within tolerance on 2-4 taps per phase, stride 1
    and 2, ragged widths and multi-row / multi-image tiles, on conv4 and conv9 with and without
    the in-kernel feed, and close to the one-tap-per-MMA kernel."""
    from paper_2306_14316_b200 import _lib

    monkeypatch.setenv("IM2WIN_PHASE", "2")
    cases = [(3, 64, 17, 19, 64, 7, 7, 2), (1, 64, 23, 9, 64, 3, 3, 2), (2, 32, 30, 31, 48, 5, 5, 2),
             (5, 32, 8, 8, 64, 3, 3, 1), (2, 40, 12, 13, 64, 3, 3, 1), (1, 64, 140, 140, 64, 7, 7, 2),
             (7, 64, 6, 7, 33, 3, 3, 1), (2, 64, 20, 21, 64, 7, 7, 1)]  # (last: 7 taps, no pairs)
    for (n, c, h, w, co, hf, wf, s) in cases:
        rng = np.random.default_rng(n * 100 + h + wf)
        if (wf + s - 1) // s > 4:  # tap pairs cover 2-4 taps per phase: the plain kernel runs
            monkeypatch.setenv("IM2WIN_PHASE_TN2", "2")
            out = pkg.conv_im2win_opt(inp := rng.standard_normal((n, c, h, w), dtype=np.float32),
                                      flt := rng.standard_normal((co, c, hf, wf), dtype=np.float32),
                                      pkg.ConvParams(c, co, hf, wf, s), variant=variant, tc_path="fused").numpy()
            assert "tap pairs" not in _lib.last_kernel()
            assert pkg.normalized_max_diff(out, orc.conv_direct(inp, flt, s)) <= TC_TOL[variant]
            continue
        inp = rng.standard_normal((n, c, h, w), dtype=np.float32)
        flt = rng.standard_normal((co, c, hf, wf), dtype=np.float32)
        ref = orc.conv_direct(inp, flt, s)
        params = pkg.ConvParams(c, co, hf, wf, s)
        monkeypatch.setenv("IM2WIN_PHASE_TN2", "2")
        out2 = pkg.conv_im2win_opt(inp, flt, params, variant=variant, tc_path="fused").numpy()
        assert "tap pairs" in _lib.last_kernel(), (n, c, h, w, _lib.last_kernel())
        monkeypatch.setenv("IM2WIN_PHASE_TN2", "0")
        out0 = pkg.conv_im2win_opt(inp, flt, params, variant=variant, tc_path="fused").numpy()
        assert pkg.normalized_max_diff(out2, ref) <= TC_TOL[variant], (n, c, h, w, co, hf, wf, s)
        assert pkg.normalized_max_diff(out2, out0) <= TC_TOL[variant] / 2, (n, c, h, w, co, hf, wf, s)
    monkeypatch.setenv("IM2WIN_PHASE_TN2", "2")
    for name in ("conv4", "conv9"):
        g = layer_goldens[name]
        cfg = replace(BENCHMARKS[name], batch=g["batch"], seed=g["seed"])
        inp, flt = make_inputs(cfg)
        ref = orc.conv_direct(inp, flt, cfg.stride)
        for feed in ("0", "2"):
            monkeypatch.setenv("IM2WIN_FEED", feed)
            out = pkg.conv_im2win_opt(inp, flt, cfg.params, variant=variant).numpy()
            assert "tap pairs" in _lib.last_kernel(), (name, feed)
            assert pkg.normalized_max_diff(out, ref) <= TC_TOL[variant], (name, feed)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("shape", [(2, 3, 7, 9), (3, 64, 12, 12), (2, 96, 20, 20), (1, 130, 6, 10), (2, 40, 5, 5),
                                   (1, 256, 14, 14)])
def test_nhwc_copy_exact(shape, dtype):
    """The channels-last copy feeding the fused TC kernels equals torch's permute (+ RN bf16
    rounding) bit for bit, zero padded to the 16-byte channel pitch; every kernel shape."""
    from paper_2306_14316_b200.kernels import nhwc_into, nhwc_pitch

    g = torch.Generator(device="cpu").manual_seed(sum(shape))
    x = torch.randn(shape, generator=g).to(DEV)
    v = "bf16" if dtype == torch.bfloat16 else "tf32"
    n, c, h, w = shape
    cp = nhwc_pitch(c, v)
    out = torch.full((n, h, w, cp), float("nan"), dtype=dtype, device=DEV)
    nhwc_into(x, out)
    ref = torch.zeros((n, h, w, cp), dtype=dtype, device=DEV)
    ref[..., :c] = x.permute(0, 2, 3, 1).to(dtype)
    assert torch.equal(out.view(torch.int16 if dtype == torch.bfloat16 else torch.int32),
                       ref.view(torch.int16 if dtype == torch.bfloat16 else torch.int32))


def _pad_np(x, p):
    return np.pad(x, ((0, 0), (0, 0), (p, p), (p, p)))


def test_native_padding_config1_golden(layer_goldens):
    """Config 1 (pad 1) with the padding done inside the transform gives the reference's
    bits for the explicitly pre-padded input (golden checksum cfg1-pad1)."""
    padded, flt = make_config1_inputs(0)
    inp = np.ascontiguousarray(padded[:, :, 1:57, 1:57])
    params = pkg.ConvParams(64, 64, 3, 3, 1, pad=1)
    out = pkg.conv_im2win_opt(inp, flt, params)
    assert orc.checksum(out.numpy()) == layer_goldens["cfg1-pad1"]["out_sha"]
    host = pkg.conv_im2win_opt_host(inp, flt, params)
    assert orc.checksum(host.numpy()) == layer_goldens["cfg1-pad1"]["out_sha"]


@pytest.mark.parametrize("case", [(2, 3, 9, 11, 4, 3, 3, 1, 1), (1, 5, 7, 6, 3, 3, 2, 2, 2), (3, 2, 5, 5, 2, 2, 2, 1, 3),
                                  (1, 4, 12, 13, 5, 7, 7, 2, 3), (2, 3, 6, 8, 2, 11, 11, 4, 5),
                                  (1, 64, 56, 56, 8, 3, 3, 1, 1), (1, 16, 20, 17, 4, 5, 5, 2, 4)])
def test_native_padding_transform_and_conv(case):
    """Padded transform == transform of the explicitly padded input (bitwise, incl. pad >= Hf:
    all-zero window rows); fp32-exact conv == the oracle on the padded input (bitwise)."""
    n, c, h, w, co, hf, wf, s, p = case
    rng = np.random.default_rng(sum(case))
    inp = rng.standard_normal((n, c, h, w), dtype=np.float32)
    flt = rng.standard_normal((co, c, hf, wf), dtype=np.float32)
    params = pkg.ConvParams(c, co, hf, wf, s, pad=p)
    win = pkg.im2win(inp, params)
    ref_win = orc.im2win_fill(_pad_np(inp, p), hf, wf, s)
    assert bits_equal(win.data.cpu().numpy(), ref_win), case
    out = pkg.conv_im2win_opt(inp, flt, params)
    assert bits_equal_nan_as_class(out.numpy(), orc.conv_direct(_pad_np(inp, p), flt, s)), case


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
def test_native_padding_tensor_cores(variant):
    """TC variants with padding: the channels-last copy writes zero borders, every fused kernel
    and the gather path stay within tolerance; the host pipeline matches the device path."""
    cases = [(2, 64, 28, 28, 64, 3, 3, 1, 1), (1, 64, 30, 30, 64, 7, 7, 2, 3), (2, 3, 32, 32, 64, 3, 3, 1, 1),
             (1, 96, 12, 12, 128, 5, 5, 1, 2)]
    for (n, c, h, w, co, hf, wf, s, p) in cases:
        rng = np.random.default_rng(h * 7 + p)
        inp = rng.standard_normal((n, c, h, w), dtype=np.float32)
        flt = rng.standard_normal((co, c, hf, wf), dtype=np.float32)
        params = pkg.ConvParams(c, co, hf, wf, s, pad=p)
        ref = orc.conv_direct(_pad_np(inp, p), flt, s)
        paths = ("fused", "gather") + (("direct",) if c <= 16 else ())
        for path in paths:
            out = pkg.conv_im2win_opt(inp, flt, params, variant=variant, tc_path=path).numpy()
            assert pkg.normalized_max_diff(out, ref) <= TC_TOL[variant], (n, c, h, w, p, path)
        dev = pkg.conv_im2win_opt(inp, flt, params, variant=variant).numpy()
        host = pkg.conv_im2win_opt_host(inp, flt, params, variant=variant, chunk_images=1).numpy()
        assert bits_equal(host, dev)
    with pytest.raises(ValueError):
        pkg.conv_im2win_opt(np.zeros((1, 8, 8, 8), np.float32), np.zeros((8, 8, 3, 3), np.float32),
                            pkg.ConvParams(8, 8, 3, 3, 1, pad=1), variant=variant, tc_path="cl")


def test_host_batch_api_order_and_bits():
    """The batch host API returns results in job order, bit-identical to one-by-one calls."""
    jobs = []
    for i, name in enumerate(["conv7", "conv12", "conv4", "conv9"]):
        cfg = replace(BENCHMARKS[name], batch=2 + i % 2, seed=60 + i)
        inp, flt = make_inputs(cfg)
        jobs.append((inp, flt, cfg.params))
    outs = pkg.conv_im2win_opt_host_batch(jobs)
    for (inp, flt, params), out in zip(jobs, outs):
        assert bits_equal(out.numpy(), pkg.conv_im2win_opt(inp, flt, params).numpy())


@pytest.mark.parametrize("variant", pkg.VARIANTS)
def test_captured_conv_replays_bitwise(variant):
    """CapturedConv (CUDA-graph replay) equals conv_im2win_opt bit for bit, for new inputs and
    a new filter on every replay, including a padded geometry and a few-channel layer (conv2:
    the direct TC kernel for TF32/BF16)."""
    for name, pad in (("conv10", 0), ("conv9", 1), ("conv2", 0)):
        cfg = replace(BENCHMARKS[name], batch=3)
        params = pkg.ConvParams(cfg.c_in, cfg.c_out, cfg.h_f, cfg.w_f, cfg.stride, pad=pad)
        cap = pkg.CapturedConv((3, cfg.c_in, cfg.h_in, cfg.w_in), params, variant=variant)
        for seed in (1, 2):
            inp, flt = make_inputs(replace(cfg, seed=seed))
            got = cap(torch.from_numpy(inp).to(DEV), torch.from_numpy(flt).to(DEV)).numpy()
            ref = pkg.conv_im2win_opt(inp, flt, params, variant=variant).numpy()
            assert bits_equal(got, ref), (name, pad, seed)


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
def test_tc_direct_layers(variant, layer_goldens):
    """The in-SM im2win tensor-core kernel on every few-channel benchmark layer (conv1-3, conv7)."""
    for name in ("conv1", "conv2", "conv3", "conv7"):
        g = layer_goldens[name]
        cfg = replace(BENCHMARKS[name], batch=g["batch"], seed=g["seed"])
        inp, flt = make_inputs(cfg)
        ref = orc.conv_direct(inp, flt, cfg.stride)
        out = pkg.conv_im2win_opt(inp, flt, cfg.params, variant=variant, tc_path="direct").numpy()
        assert pkg.normalized_max_diff(out, ref) <= TC_TOL[variant], name
        from paper_2306_14316_b200 import _lib
        assert "conv_tc_direct_kernel" in _lib.last_kernel()


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
def test_tc_direct_geometries(variant):
    """Direct kernel on ragged geometries: C 1..16, strides 1-4, filters up to 11x11, padding,
    multi-row tiles, split rows (w_out > 128), one image and odd batch counts."""
    cases = [(1, 1, 9, 7, 16, 3, 3, 1, 0), (3, 3, 40, 300, 64, 5, 5, 2, 2), (2, 4, 31, 33, 96, 11, 11, 4, 0),
             (2, 8, 17, 17, 128, 7, 7, 2, 3), (1, 16, 12, 12, 256, 3, 3, 1, 1), (5, 3, 20, 20, 64, 3, 3, 1, 1),
             (1, 2, 8, 140, 32, 1, 1, 1, 0)]
    for (n, c, h, w, co, hf, wf, s, p) in cases:
        rng = np.random.default_rng(n + c + h + w)
        inp = rng.standard_normal((n, c, h, w), dtype=np.float32)
        flt = rng.standard_normal((co, c, hf, wf), dtype=np.float32)
        ref = orc.conv_direct(_pad_np(inp, p), flt, s)
        params = pkg.ConvParams(c, co, hf, wf, s, pad=p)
        if not pkg.kernels.direct_supported(inp.shape, params, variant):
            # tf32 with a large window: the resident filter would not fit; auto uses the fused path
            assert variant == "tf32", (n, c, h, w, co, hf, wf, s, p)
            with pytest.raises(ValueError):
                pkg.conv_im2win_opt(inp, flt, params, variant=variant, tc_path="direct")
            out = pkg.conv_im2win_opt(inp, flt, params, variant=variant).numpy()
        else:
            out = pkg.conv_im2win_opt(inp, flt, params, variant=variant, tc_path="direct").numpy()
        assert pkg.normalized_max_diff(out, ref) <= TC_TOL[variant], (n, c, h, w, co, hf, wf, s, p)


def test_host_pipeline_device_list_slices():
    """devices=[...] splits the batch into per-device slices submitted concurrently; with the one
    GPU of this box listed several times the slices share it and the result is still the
    single-call result bit for bit (ragged slices included)."""
    cfg = replace(BENCHMARKS["conv9"], batch=7, seed=12)
    inp, flt = make_inputs(cfg)
    ref = pkg.conv_im2win_opt_host(inp, flt, cfg.params).numpy()
    for devs in ([0, 0], [0, 0, 0], ["cuda:0"] * 4):
        got = pkg.conv_im2win_opt_host(inp, flt, cfg.params, devices=devs, chunk_images=1).numpy()
        assert bits_equal(got, ref), devs
    outs = pkg.conv_im2win_opt_host_batch([(inp, flt, cfg.params)], devices=[0, 0])
    assert bits_equal(outs[0].numpy(), ref)


def test_memory_budget_refusal():
    """run_bench refuses a configuration that cannot fit before allocating anything
    (reference bench.py:179-183, test_bench.py:114-120), with the byte counts."""
    cfg = replace(BENCHMARKS["conv4"], batch=100_000)
    with pytest.raises(pkg.MemoryBudgetError) as e:
        pkg.run_bench(replace(cfg, repeats=1))
    assert e.value.required_bytes > e.value.available_bytes > 0


@pytest.mark.parametrize("pad", [0, 2])
def test_unaligned_and_degenerate_inputs(pad):
    """Operands at a 4-byte offset (the transform's 16-byte TMA path cannot take them: the
    legacy kernel / an aligned copy is used), one-pixel outputs (filter = padded input) and a
    single image all give the oracle's bits."""
    rng = np.random.default_rng(77 + pad)
    base = torch.from_numpy(rng.standard_normal(1 + 2 * 4 * 9 * 11, dtype=np.float32)).to(DEV)
    x = base[1:].view(2, 4, 9, 11)  # data_ptr % 16 == 4
    assert x.data_ptr() % 16 != 0
    flt = rng.standard_normal((5, 4, 3, 3), dtype=np.float32)
    params = pkg.ConvParams(4, 5, 3, 3, 2, pad=pad)
    xn = x.cpu().numpy()
    win = pkg.im2win(x, params)
    assert bits_equal(win.data.cpu().numpy(), orc.im2win_fill(_pad_np(xn, pad), 3, 3, 2))
    out = pkg.conv_im2win_opt(x, torch.from_numpy(flt).to(DEV), params)
    assert bits_equal_nan_as_class(out.numpy(), orc.conv_direct(_pad_np(xn, pad), flt, 2))
    # filter as large as the (padded) input: one output pixel per image and channel
    h = 7 - 2 * pad
    xi = rng.standard_normal((1, 3, h, h), dtype=np.float32)
    fi = rng.standard_normal((2, 3, 7, 7), dtype=np.float32)
    p1 = pkg.ConvParams(3, 2, 7, 7, 1, pad=pad)
    o1 = pkg.conv_im2win_opt(xi, fi, p1)
    assert o1.dims == (1, 2, 1, 1)
    assert bits_equal_nan_as_class(o1.numpy(), orc.conv_direct(_pad_np(xi, pad), fi, 1))


@pytest.mark.parametrize("group", ["1", "3", "5"])
def test_tc_fused_tile_groups(group, layer_goldens, monkeypatch):
    """The generic fused kernel's tile walk (runs of `group` consecutive tiles per CTA) covers
    every tile exactly once: conv7 (two pieces per output row) and a ragged geometry."""
    monkeypatch.setenv("IM2WIN_TILE_GROUP", group)
    monkeypatch.setenv("IM2WIN_PHASE", "0")
    monkeypatch.setenv("IM2WIN_SHIFT", "0")
    g = layer_goldens["conv7"]
    cfg = replace(BENCHMARKS["conv7"], batch=g["batch"], seed=g["seed"])
    inp, flt = make_inputs(cfg)
    ref = orc.conv_direct(inp, flt, cfg.stride)
    out = pkg.conv_im2win_opt(inp, flt, cfg.params, variant="bf16", tc_path="fused").numpy()
    assert pkg.normalized_max_diff(out, ref) <= TC_TOL["bf16"]
    rng = np.random.default_rng(int(group))
    inp = rng.standard_normal((3, 8, 9, 300), dtype=np.float32)
    flt = rng.standard_normal((40, 8, 3, 3), dtype=np.float32)
    ref = orc.conv_direct(inp, flt, 1)
    for v in ("tf32", "bf16"):
        out = pkg.conv_im2win_opt(inp, flt, pkg.ConvParams(8, 40, 3, 3, 1), variant=v, tc_path="fused").numpy()
        assert pkg.normalized_max_diff(out, ref) <= TC_TOL[v], v


@pytest.mark.parametrize("variant", ["fp32-exact", "fp32-fma"])
def test_simt_smallk_persistent_kernel(variant):
    """The persistent small-K SIMT kernel (library choice for K <= 64, Co <= 64 with enough
    tiles: conv7) gives the bits of the tiled kernel (explicit 64x256 plan) and of the oracle,
    including special values, a ragged last tile and odd K (padded k never computed)."""
    from paper_2306_14316_b200 import _lib
    for (n, c, h, w, co, hf, wf) in [(16, 3, 224, 224, 64, 3, 3), (20, 5, 161, 203, 40, 3, 3), (32, 7, 130, 150, 64, 2, 3),
                                          (20, 1, 180, 180, 32, 4, 4), (14, 4, 212, 212, 64, 4, 4)]:
        rng = np.random.default_rng(n * 100 + c)
        inp = rng.standard_normal((n, c, h, w), dtype=np.float32)
        inp[0, 0, 0, :5] = [np.inf, -np.inf, np.nan, 0.0, -0.0]
        flt = rng.standard_normal((co, c, hf, wf), dtype=np.float32)
        params = pkg.ConvParams(c, co, hf, wf, 1)
        win = pkg.im2win(torch.from_numpy(inp).to(DEV), params)
        out = pkg.compute_from_windows_opt(win, torch.from_numpy(flt).to(DEV), params, variant=variant)
        assert "smallk" in _lib.last_kernel(), _lib.last_kernel()
        tiled = pkg.compute_from_windows_opt(win, torch.from_numpy(flt).to(DEV), params,
                                             pkg.TilePlan(64, 256, 8, 8, 8), variant=variant)
        assert bits_equal_nan_as_class(out.numpy(), tiled.numpy()), (n, c, h, w)
        if variant == "fp32-exact":
            for i in (0, n - 1):
                ref = orc.conv_direct(inp[i:i + 1], flt, 1)
                assert bits_equal_nan_as_class(out.data[i:i + 1].cpu().numpy(), ref), (n, c, h, w, i)


# ---------------------------------------------------------------- full-size sampled parity
def _device_inputs(cfg, seed):
    g = torch.Generator(device=DEV).manual_seed(seed)
    x = torch.randn((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), device=DEV, generator=g)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=DEV, generator=g)
    return x, f


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
@pytest.mark.parametrize("name", ["conv9", "conv10", "conv11", "conv12"])
def test_tc_config4_n1024_sampled_images(name, variant):
    """BASELINE config 4: the ResNet-50 3x3 layers at N=1024 through the production TC path;
    images are independent (reference.py:78-90), so sampled images vs the oracle pin the batch."""
    cfg = replace(BENCHMARKS[name], batch=1024)
    x, f = _device_inputs(cfg, 41)
    out = pkg.conv_im2win_opt(x, f, cfg.params, variant=variant).data
    fh = f.cpu().numpy()
    for i in (0, 333, 1023):
        xi = x[i:i + 1].cpu().numpy()
        ref = orc.conv_direct(xi, fh, cfg.stride)
        got = out[i:i + 1].cpu().numpy()
        assert pkg.normalized_max_diff(got, ref) <= TC_TOL[variant], (name, i)
        assert _tc_elementwise_ok(got, ref, xi, fh, cfg.stride, variant), (name, i)


@pytest.mark.parametrize("name", list(BENCHMARKS))
def test_all_layers_n256_sampled_images(name):
    """BASELINE config 5 per-GPU shard (N=256 of 2048 over 8 GPUs), every layer: FP32-exact
    bitwise and TF32/BF16 within tolerance on sampled images against the oracle."""
    cfg = replace(BENCHMARKS[name], batch=256)
    x, f = _device_inputs(cfg, 43)
    fh = f.cpu().numpy()
    outs = {v: pkg.conv_im2win_opt(x, f, cfg.params, variant=v).data for v in ("fp32-exact", "tf32", "bf16")}
    for i in (0, 129, 255):
        xi = x[i:i + 1].cpu().numpy()
        ref = orc.conv_direct(xi, fh, cfg.stride)
        assert bits_equal(outs["fp32-exact"][i:i + 1].cpu().numpy(), ref), (name, i)
        for v in ("tf32", "bf16"):
            assert pkg.normalized_max_diff(outs[v][i:i + 1].cpu().numpy(), ref) <= TC_TOL[v], (name, v, i)


# ---------------------------------------------------------------- im2win_gather (layouts.py:98-105)
def test_im2win_gather_fig1():
    """Fig. 1: 3x3x3 input, 2x2 filter, stride 1 (pkg/tests/test_layouts.py:218-232)."""
    img = np.arange(1, 28, dtype=np.float32).reshape(1, 3, 3, 3)
    p = pkg.ConvParams(3, 1, 2, 2, 1)
    w = pkg.im2win(torch.from_numpy(img).to(DEV), p)
    assert pkg.im2win_gather(w, 0, 0, 0, 0, 0, 0) == img[0, 0, 0, 0]
    for r in range(3):
        got = [[pkg.im2win_gather(w, 0, r, 0, fh, fw, 1) for fw in range(2)] for fh in range(2)]
        assert got == img[0, r, 0:2, 1:3].tolist()
    with pytest.raises(IndexError):
        pkg.im2win_gather(w, 0, 0, 0, 2, 0, 0)
    with pytest.raises(IndexError):
        pkg.im2win_gather(w, 1, 0, 0, 0, 0, 0)


def test_im2win_gather_matches_direct_reads():
    """10^4 random reads equal the input element they stand for (pkg/tests/test_layouts.py:235-249)."""
    rng = np.random.default_rng(11)
    for (n, c, h, w, hf, wf, s) in ((2, 3, 17, 19, 3, 5, 2), (1, 4, 12, 12, 4, 4, 1), (3, 2, 23, 20, 7, 3, 3)):
        inp = rng.standard_normal((n, c, h, w), dtype=np.float32)
        p = pkg.ConvParams(c, 1, hf, wf, s)
        win = pkg.im2win(torch.from_numpy(inp).to(DEV), p)
        for _ in range(3400):
            i_n, i_c = int(rng.integers(0, win.n)), int(rng.integers(0, win.c_in))
            o_h, o_w = int(rng.integers(0, win.h_out)), int(rng.integers(0, win.w_out))
            f_h, f_w = int(rng.integers(0, hf)), int(rng.integers(0, wf))
            assert pkg.im2win_gather(win, i_n, i_c, o_h, f_h, f_w, o_w) == inp[i_n, i_c, o_h * s + f_h, o_w * s + f_w]


# ---------------------------------------------------------------- harness drop-in (bench.py:43-59, 226, 342)
def test_reference_harness_call_and_search_plan(layer_goldens):
    """BASELINE.md's own call against this package, and search_plan over the compiled tiles."""
    rec = pkg.run_bench(replace(BENCHMARKS["conv9"], batch=8, repeats=3, algorithm="im2win-opt"))
    assert rec.repeats == 3 and rec.algorithm == "im2win-opt" and rec.variant == "-" and rec.tflops > 0
    # the record's checksum is the reference's: same seeded numpy operands (bench.py:152-159)
    g = layer_goldens["conv9"]
    cfg = replace(BENCHMARKS["conv9"], batch=g["batch"], seed=g["seed"])
    assert pkg.run_bench(replace(cfg, repeats=1)).checksum == g["out_sha"]
    alias = pkg.run_bench(replace(cfg, repeats=1, algorithm="im2col-gemm"), "baseline")
    assert alias.algorithm == "im2col-gemm" and alias.variant == "baseline"
    from paper_2306_14316_b200.harness import DEFAULT_SEARCH_GRID, search_plan
    res = search_plan(replace(cfg, batch=4))
    assert len(res) == len(DEFAULT_SEARCH_GRID)
    assert [t for _, t in res] == sorted(t for _, t in res)
    assert all(isinstance(p, pkg.TilePlan) for p, _ in res)
    # reference-grid entries that name no compiled tile are skipped
    assert [p for p, _ in search_plan(replace(cfg, batch=2), grid=((16, 16, 4), (64, 64, 16)))] == [
        pkg.TilePlan(64, 64, 16, 4, 4)]
    abl = pkg.run_ablation(replace(cfg, batch=4, repeats=1))
    assert len({r.checksum for r in abl}) == 1


def _feed_vs_copy(inp, flt, params, variant, monkeypatch):
    """conv_im2win_opt with the in-kernel feed forced vs with the copy kernel forced: same bits."""
    monkeypatch.setenv("IM2WIN_FEED", "2")
    fed = pkg.conv_im2win_opt(inp, flt, params, variant=variant, tc_path="fused").numpy()
    monkeypatch.setenv("IM2WIN_FEED", "0")
    copied = pkg.conv_im2win_opt(inp, flt, params, variant=variant, tc_path="fused").numpy()
    monkeypatch.delenv("IM2WIN_FEED")
    return fed, copied


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
@pytest.mark.parametrize("select", ["auto", "phase", "shift", "generic"])
def test_tc_feed_bitwise_all_layers(select, variant, layer_goldens, monkeypatch):
    """The channels-last copy produced by the conv kernel's own feed warps (im2win_conv_fused_nchw)
    gives the same bits as the separate copy kernel, for every TMA-fed kernel and layer; and the
    result is within the stated tolerance of the reference golden's oracle."""
    env = {"auto": ("1", "1"), "phase": ("2", "0"), "shift": ("0", "2"), "generic": ("0", "0")}[select]
    monkeypatch.setenv("IM2WIN_PHASE", env[0])
    monkeypatch.setenv("IM2WIN_SHIFT", env[1])
    for name in BENCHMARKS:
        g = layer_goldens[name]
        cfg = replace(BENCHMARKS[name], batch=g["batch"], seed=g["seed"])
        inp, flt = make_inputs(cfg)
        fed, copied = _feed_vs_copy(inp, flt, cfg.params, variant, monkeypatch)
        assert bits_equal(fed, copied), (name, select)
        assert pkg.normalized_max_diff(fed, orc.conv_direct(inp, flt, cfg.stride)) <= TC_TOL[variant], (name, select)


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
def test_tc_feed_ragged_geometries(variant, monkeypatch):
    """Feed units on ragged shapes: pixel counts not a multiple of the unit's 64/128 pixels, channel
    counts not a multiple of the 8/16-channel group (and below the 16-byte pitch), one image, many
    images smaller than a unit, the phase kernel's multi-image tiles."""
    cases = [(3, 64, 17, 19, 64, 7, 7, 2), (2, 40, 12, 13, 128, 3, 3, 1), (1, 3, 30, 33, 64, 3, 3, 1),
             (9, 72, 7, 7, 96, 3, 3, 1), (4, 130, 9, 10, 256, 3, 3, 1), (1, 64, 140, 140, 64, 7, 7, 2),
             (7, 16, 5, 6, 64, 3, 3, 1)]
    for (n, c, h, w, co, hf, wf, s) in cases:
        rng = np.random.default_rng(n * 1000 + h + c)
        inp = rng.standard_normal((n, c, h, w), dtype=np.float32)
        flt = rng.standard_normal((co, c, hf, wf), dtype=np.float32)
        params = pkg.ConvParams(c, co, hf, wf, s)
        fed, copied = _feed_vs_copy(inp, flt, params, variant, monkeypatch)
        assert bits_equal(fed, copied), (n, c, h, w, co, hf, wf, s)
        assert pkg.normalized_max_diff(fed, orc.conv_direct(inp, flt, s)) <= TC_TOL[variant], (n, c, h, w)


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
def test_tc_feed_conv4_n128_sampled_images(variant):
    """The auto rule feeds conv4 (output/input elements 0.24): at N=128 every sampled image
    matches the oracle within tolerance (images are independent, reference.py:78-90)."""
    cfg = replace(BENCHMARKS["conv4"], batch=128)
    g = torch.Generator(device=DEV).manual_seed(44)
    x = torch.randn((128, cfg.c_in, cfg.h_in, cfg.w_in), device=DEV, generator=g)
    f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=DEV, generator=g)
    out = pkg.conv_im2win_opt(x, f, cfg.params, variant=variant)
    from paper_2306_14316_b200 import _lib

    assert "phase" in _lib.last_kernel()
    fn = f.cpu().numpy()
    for i in (0, 1, 63, 127):
        ref = orc.conv_direct(x[i:i + 1].cpu().numpy(), fn, cfg.stride)
        assert pkg.normalized_max_diff(out.data[i:i + 1].cpu().numpy(), ref) <= TC_TOL[variant], i


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
def test_tc_phase_cta_pair(variant, layer_goldens, monkeypatch):
    """The phase kernel on CTA pairs (cta_group::2, UMMA M = 256, filter halves per CTA,
    IM2WIN_PAIR=1) is within tolerance on every layer it takes and on ragged geometries (odd
    pixel-tile counts leave the second CTA's tiles empty), with and without the feed."""
    monkeypatch.setenv("IM2WIN_PAIR", "1")
    monkeypatch.setenv("IM2WIN_PHASE", "2")
    monkeypatch.setenv("IM2WIN_SHIFT", "0")
    from paper_2306_14316_b200 import _lib

    for name in BENCHMARKS:
        g = layer_goldens[name]
        cfg = replace(BENCHMARKS[name], batch=g["batch"], seed=g["seed"])
        inp, flt = make_inputs(cfg)
        ref = orc.conv_direct(inp, flt, cfg.stride)
        for feed in ("0", "2"):
            monkeypatch.setenv("IM2WIN_FEED", feed)
            out = pkg.conv_im2win_opt(inp, flt, cfg.params, variant=variant, tc_path="fused").numpy()
            assert pkg.normalized_max_diff(out, ref) <= TC_TOL[variant], (name, feed)
    cases = [(3, 64, 17, 19, 64, 7, 7, 2), (1, 64, 23, 9, 64, 3, 3, 2), (2, 40, 12, 13, 128, 3, 3, 1),
             (5, 32, 8, 8, 64, 5, 5, 1)]
    seen = set()
    for (n, c, h, w, co, hf, wf, s) in cases:
        rng = np.random.default_rng(n * 1000 + h)
        inp = rng.standard_normal((n, c, h, w), dtype=np.float32)
        flt = rng.standard_normal((co, c, hf, wf), dtype=np.float32)
        out = pkg.conv_im2win_opt(inp, flt, pkg.ConvParams(c, co, hf, wf, s), variant=variant,
                                  tc_path="fused").numpy()
        seen.add(_lib.last_kernel())
        assert pkg.normalized_max_diff(out, orc.conv_direct(inp, flt, s)) <= TC_TOL[variant], (n, c, h, w)
    assert any("CTA pair" in k for k in seen), seen


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
def test_captured_conv_with_feed(variant, monkeypatch):
    """CapturedConv records the one-call fused path with the in-kernel feed (a cooperative
    launch plus the counter memset) and replays it bit-identically to the eager call."""
    monkeypatch.setenv("IM2WIN_FEED", "2")
    params = pkg.ConvParams(64, 64, 7, 7, 2)
    g = torch.Generator(device=DEV).manual_seed(3)
    x = torch.randn((3, 64, 40, 44), device=DEV, generator=g)
    f = torch.randn((64, 64, 7, 7), device=DEV, generator=g)
    cc = pkg.CapturedConv(x.shape, params, f, variant=variant)
    eager = pkg.conv_im2win_opt(x, f, params, variant=variant).numpy()
    for _ in range(2):
        got = cc(x).numpy()
        assert bits_equal(got, eager)
    x2 = torch.randn_like(x)
    assert bits_equal(cc(x2).numpy(), pkg.conv_im2win_opt(x2, f, params, variant=variant).numpy())


@pytest.mark.parametrize("variant", ["fp32-exact", "fp32-fma"])
def test_fp32_window_budget_chunks_bitwise(variant, monkeypatch, layer_goldens):
    """With Ĩ above the window budget conv_im2win_opt transforms and convolves image chunks
    through one reused Ĩ buffer: same bits as the full-batch call (ragged last chunk, padding),
    and the reference goldens still match."""
    for name, n in (("conv9", 19), ("conv3", 9), ("conv12", 17)):
        cfg = replace(BENCHMARKS[name], batch=n, seed=5)
        inp, flt = make_inputs(cfg)
        x = torch.from_numpy(inp).to(DEV)
        monkeypatch.setenv("IM2WIN_WINDOW_BUDGET", "0")
        full = pkg.conv_im2win_opt(x, flt, cfg.params, variant=variant).numpy()
        monkeypatch.setenv("IM2WIN_WINDOW_BUDGET", "1")  # forces chunks of 8 images
        chunked = pkg.conv_im2win_opt(x, flt, cfg.params, variant=variant).numpy()
        assert bits_equal(chunked, full), name
    monkeypatch.setenv("IM2WIN_WINDOW_BUDGET", "1")
    params = pkg.ConvParams(3, 8, 3, 3, 1, pad=1)
    rng = np.random.default_rng(2)
    inp = rng.standard_normal((11, 3, 13, 10), dtype=np.float32)
    flt = rng.standard_normal((8, 3, 3, 3), dtype=np.float32)
    chunked = pkg.conv_im2win_opt(inp, flt, params, variant=variant).numpy()
    monkeypatch.setenv("IM2WIN_WINDOW_BUDGET", "0")
    assert bits_equal(chunked, pkg.conv_im2win_opt(inp, flt, params, variant=variant).numpy())
    if variant == "fp32-exact":
        g = layer_goldens["conv9"]
        cfg = replace(BENCHMARKS["conv9"], batch=g["batch"], seed=g["seed"])
        inp, flt = make_inputs(cfg)
        monkeypatch.setenv("IM2WIN_WINDOW_BUDGET", "1")
        out = pkg.conv_im2win_opt(inp, flt, cfg.params).numpy()
        assert orc.checksum(out) == g["out_sha"]


def test_nchw_direct_all_tiles_and_toggles_bitwise(small_cases):
    """The FP32 kernels gathering windows straight from NCHW (im2win_conv_nchw_f32, the default
    of conv_im2win_opt) give the reference's bits for every compiled CTA tile and toggle, on Fig. 1,
    the special-values case, the 1x1 identity and the random geometries."""
    from paper_2306_14316_b200.kernels import conv_nchw_into

    names = ["fig1", "special", "identity1x1"] + [f"rand{i:03d}" for i in range(0, 200, 5)]
    for name in names:
        c = small_cases[name]
        params = _params(c)
        inp = torch.from_numpy(c["inp"]).to(DEV)
        flt = torch.from_numpy(c["flt"]).to(DEV)
        plans = [None]
        for (bm, bn) in pkg.plan.SIMT_TILES:
            for vec in (True, False):
                for pf in (True, False):
                    plans.append(pkg.TilePlan(bm, bn, 8, 8, 8, vectorized_load=vec, prefetch_double_buffer=pf))
        plans += [pkg.TilePlan(bm, bn, 8, 4, 4) for (bm, bn) in pkg.plan.SIMT_TILES_MT4]
        for plan in plans:
            out = torch.full(c["out"].shape, float("nan"), device=DEV)
            conv_nchw_into(inp, flt, out, params, plan)
            assert bits_equal_nan_as_class(out.cpu().numpy(), c["out"]), (name, plan)


@pytest.mark.parametrize("variant", ["fp32-exact", "fp32-fma"])
def test_nchw_direct_equals_window_path_all_layers(variant, monkeypatch, layer_goldens):
    """conv_im2win_opt (NCHW-direct) == im2win + compute_from_windows_opt bit for bit on all 12
    layers (the golden checksums for fp32-exact), and on the small-K persistent kernel's shapes."""
    for name in BENCHMARKS:
        g = layer_goldens[name]
        cfg = replace(BENCHMARKS[name], batch=g["batch"], seed=g["seed"])
        inp, flt = make_inputs(cfg)
        direct = pkg.conv_im2win_opt(inp, flt, cfg.params, variant=variant).numpy()
        windows = pkg.compute_from_windows_opt(pkg.im2win(inp, cfg.params), flt, cfg.params,
                                               variant=variant).numpy()
        assert bits_equal(direct, windows), name
        if variant == "fp32-exact":
            assert orc.checksum(direct) == g["out_sha"], name
    monkeypatch.setenv("IM2WIN_FP32_PATH", "windows")
    g = layer_goldens["conv9"]
    cfg = replace(BENCHMARKS["conv9"], batch=g["batch"], seed=g["seed"])
    inp, flt = make_inputs(cfg)
    assert bits_equal(pkg.conv_im2win_opt(inp, flt, cfg.params, variant=variant).numpy(),
                      pkg.compute_from_windows_opt(pkg.im2win(inp, cfg.params), flt, cfg.params,
                                                   variant=variant).numpy())


def test_nchw_direct_large_batch_sampled_images():
    """NCHW-direct FP32-exact at N=128 (conv4 and conv8: K in whole slabs, the predicate-free
    gather; conv3: padded last K slab computed over its real rows; conv7 small-K, conv12 4x4 tiles,
    conv1 96-wide tiles and tail split): sampled images bitwise equal to the oracle."""
    for name in ("conv4", "conv8", "conv3", "conv7", "conv12", "conv1"):
        cfg = replace(BENCHMARKS[name], batch=128)
        g = torch.Generator(device=DEV).manual_seed(77)
        x = torch.randn((128, cfg.c_in, cfg.h_in, cfg.w_in), device=DEV, generator=g)
        f = torch.randn((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), device=DEV, generator=g)
        out = pkg.conv_im2win_opt(x, f, cfg.params)
        fn = f.cpu().numpy()
        for i in (0, 77, 127):
            ref = orc.conv_direct(x[i:i + 1].cpu().numpy(), fn, cfg.stride)
            assert bits_equal(out.data[i:i + 1].cpu().numpy(), ref), (name, i)


@pytest.mark.parametrize("variant", ["tf32", "bf16"])
def test_tc_fused_64byte_rows(variant, monkeypatch, layer_goldens):
    """The fused kernel with 64-byte K rows (window rows Wf * C_pad that fit in 64 bytes: conv7 and
    few-channel odd shapes) gives the same bits as 128-byte rows (the extra K of those is zero
    padding) and stays within tolerance of the oracle."""
    from paper_2306_14316_b200 import _lib

    g = layer_goldens["conv7"]
    cfg = replace(BENCHMARKS["conv7"], batch=g["batch"], seed=g["seed"])
    cases = [(make_inputs(cfg), cfg.params)]
    for (n, c, h, w, co, hf, wf, s) in [(3, 3, 17, 21, 64, 3, 3, 1), (2, 2, 12, 13, 96, 3, 3, 2),
                                        (1, 4, 30, 31, 128, 2, 2, 1), (2, 1, 9, 10, 64, 3, 5, 1)]:
        rng = np.random.default_rng(n * 100 + c)
        cases.append(((rng.standard_normal((n, c, h, w), dtype=np.float32),
                       rng.standard_normal((co, c, hf, wf), dtype=np.float32)), pkg.ConvParams(c, co, hf, wf, s)))
    for (inp, flt), params in cases:
        monkeypatch.setenv("IM2WIN_ROW64", "1")
        r64 = pkg.conv_im2win_opt(inp, flt, params, variant=variant, tc_path="fused").numpy()
        kern = _lib.last_kernel()
        monkeypatch.setenv("IM2WIN_ROW64", "0")
        r128 = pkg.conv_im2win_opt(inp, flt, params, variant=variant, tc_path="fused").numpy()
        assert bits_equal(r64, r128), (params, kern)
        assert pkg.normalized_max_diff(r64, orc.conv_direct(inp, flt, params.stride)) <= TC_TOL[variant], params
    monkeypatch.setenv("IM2WIN_ROW64", "1")
    inp, flt = cases[0][0]
    pkg.conv_im2win_opt(inp, flt, cfg.params, variant=variant, tc_path="fused")
    assert "64-byte rows" in _lib.last_kernel()


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_nhwc_copy_small_image_block_kernel(dtype, monkeypatch):
    """The channels-last copy of small images whose H*W is not a multiple of 4 (7x7: conv12) goes
    through the 32-channel block kernel: equal to the 32x32 generic kernel and to a torch
    permute + pad + cast, for odd channel counts, a channel tail, unaligned images and a border."""
    from paper_2306_14316_b200.kernels import nhwc_into

    q = 8 if dtype == torch.bfloat16 else 4
    g = torch.Generator(device=DEV).manual_seed(21)
    for (n, c, h, w, pad) in [(3, 512, 7, 7, 0), (2, 33, 5, 9, 0), (2, 9, 15, 15, 1), (1, 70, 13, 11, 0),
                              (4, 16, 3, 3, 2)]:
        x = torch.randn((n, c, h, w), device=DEV, generator=g)
        pitch = -(-c // q) * q
        got = torch.full((n, h + 2 * pad, w + 2 * pad, pitch), 7.0, device=DEV, dtype=dtype)
        ref = torch.full_like(got, 7.0)
        nhwc_into(x, got, pad)
        monkeypatch.setenv("IM2WIN_COPY_BLOCK", "0")
        nhwc_into(x, ref, pad)
        monkeypatch.delenv("IM2WIN_COPY_BLOCK")
        want = torch.zeros_like(got)
        want[:, pad:pad + h, pad:pad + w, :c] = x.permute(0, 2, 3, 1).to(dtype)
        assert torch.equal(got.view(torch.int16 if dtype == torch.bfloat16 else torch.int32),
                           ref.view(torch.int16 if dtype == torch.bfloat16 else torch.int32)), (n, c, h, w, pad)
        assert torch.equal(got.float(), want.float()), (n, c, h, w, pad)
