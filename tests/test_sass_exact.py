"""The bit-exact FP32 kernels never fuse a product into a sum (CPU test: reads the built library's SASS).

The reference rounds twice per multiply-add (optimized.py:162-165).  The kernels issue the pair as
scalar FMUL + FADD or as two packed FFMA2 -- rn(a*b) = fma(a, b, -0) and rn(c + p) = fma(c, 1, p) --
whose -0 / 1 come from kernel arguments (uniform registers in SASS).  So in every EXACT
instantiation: no scalar FFMA at all, and every FFMA2 has a uniform-register operand (the opaque
constant); an FFMA2 of three ordinary registers would be a fused a*b + c (one rounding).
"""
import re
import shutil
import subprocess
from pathlib import Path

import pytest

LIB = Path(__file__).resolve().parent.parent / "paper_2306_14316_b200" / "libim2win_sm100.so"


def _functions():
    if not LIB.exists() or shutil.which("cuobjdump") is None:
        pytest.skip("library not built or cuobjdump missing")
    out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
    funcs, name = {}, None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            name = m.group(1)
            funcs[name] = []
        elif name:
            funcs[name].append(line)
    return funcs


def _exact(name: str) -> bool:
    # conv_simt_kernel<BM, BN, BK, STAGES, EXACT, ...>: EXACT is the first bool; smallk<KP, EXACT>
    m = re.search(r"conv_simt(?:_smallk)?_kernelI(?:Li\d+E)+Lb([01])E", name)
    return bool(m and m.group(1) == "1")


def test_exact_simt_kernels_round_twice():
    funcs = {n: body for n, body in _functions().items() if "conv_simt" in n and _exact(n)}
    assert funcs, "no EXACT conv_simt instantiation found"
    packed = 0
    for name, body in funcs.items():
        for line in body:
            ins = re.search(r"\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9]+(?:\.[A-Z0-9_]+)*)\s", line)
            if not ins:
                continue
            op = ins.group(1)
            assert not op.startswith("FFMA") or op.startswith("FFMA2"), (name, line.strip())
            if op.startswith("FFMA2"):
                packed += 1
                assert re.search(r"\bUR\d+\.F32\b", line), (name, line.strip())
    assert packed > 0, "the packed exact form is not in the library"
