"""Pin the CPU oracle (oracle/) against the reference's own outputs (tests/golden/)."""

from dataclasses import replace

import numpy as np
import pytest

from conftest import bits_equal
from oracle import oracle as orc
from paper_2306_14316_b200.workloads import BENCHMARKS, make_config1_inputs, make_inputs


def test_oracle_transform_matches_reference_goldens(small_cases):
    assert len(small_cases) >= 205
    for name, c in small_cases.items():
        win = orc.im2win_fill(c["inp"], c["h_f"], c["w_f"], c["stride"], threads=2)
        assert bits_equal(win, c["win"]), name


def test_oracle_conv_matches_reference_goldens(small_cases):
    for name, c in small_cases.items():
        out = orc.conv_direct(c["inp"], c["flt"], c["stride"], threads=2)
        assert bits_equal(out, c["out"]), name
        w_out = c["out"].shape[3]
        out2 = orc.conv_from_windows(c["win"], c["flt"], c["stride"], w_out, threads=2)
        assert bits_equal(out2, c["out"]), name


def test_fig1_known_answers(small_cases):
    c = small_cases["fig1"]
    assert c["win"].shape == (1, 3, 2, 6) and c["win"].size == 36
    # column-major within a source column (test_layouts.py:126-134)
    assert c["win"][0, 0, 0].tolist() == [0, 3, 1, 4, 2, 5]
    e = small_cases["edge_cols"]["win"]
    assert 4.0 not in e and 9.0 not in e
    assert (small_cases["ones"]["out"] == 4.0).all()


@pytest.mark.parametrize("name", list(BENCHMARKS))
def test_oracle_layer_checksums(name, layer_goldens):
    g = layer_goldens[name]
    cfg = replace(BENCHMARKS[name], batch=g["batch"], seed=g["seed"])
    inp, flt = make_inputs(cfg)
    win = orc.im2win_fill(inp, cfg.h_f, cfg.w_f, cfg.stride)
    assert orc.checksum(win) == g["win_sha"]
    out = orc.conv_direct(inp, flt, cfg.stride)
    assert orc.checksum(out) == g["out_sha"]


def test_oracle_config1(layer_goldens):
    inp, flt = make_config1_inputs(0)
    out = orc.conv_direct(inp, flt, 1)
    assert orc.checksum(out) == layer_goldens["cfg1-pad1"]["out_sha"]
