import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def small_cases():
    """Golden arrays produced by the reference package (tests/golden/make_golden.py)."""
    data = np.load(GOLDEN / "small_cases.npz")
    keys = sorted({k.split("/")[0] for k in data.files})
    cases = {}
    for k in keys:
        geom = data[f"{k}/geom"]
        cases[k] = dict(inp=data[f"{k}/inp"], flt=data[f"{k}/flt"], win=data[f"{k}/win"],
                        out=data[f"{k}/out"], c_in=int(geom[0]), c_out=int(geom[1]),
                        h_f=int(geom[2]), w_f=int(geom[3]), stride=int(geom[4]))
    return cases


@pytest.fixture(scope="session")
def layer_goldens():
    return json.loads((GOLDEN / "layers.json").read_text())


def bits_equal(a, b) -> bool:
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    return a.shape == b.shape and bool((a.view(np.uint32) == b.view(np.uint32)).all())


def bits_equal_nan_as_class(a, b) -> bool:
    """Bitwise equality except that any NaN matches any NaN.

    NaN *payloads* produced by arithmetic are ISA-specific (x86 SSE propagates the
    operand's payload and makes 0xffc00000 for invalid ops; the GPU returns the
    canonical 0x7fffffff), so conv outputs compare NaN-ness, every other bit exactly.
    Pure copies (the transform) keep payloads and are compared with bits_equal.
    """
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    if not (na == nb).all():
        return False
    return bool((a.view(np.uint32)[~na] == b.view(np.uint32)[~nb]).all())
