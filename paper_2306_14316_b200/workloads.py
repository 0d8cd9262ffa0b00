"""The paper's twelve benchmark layers and seeded synthetic operands.

Mirrors winconv `bench.py`: `BenchConfig` (/root/reference/pkg/src/winconv/bench.py:43-80),
same fields and defaults
(batch, repeats, algorithm, plan, seed), `BENCHMARKS` (:88-104), `make_inputs` (:152-159, numpy PCG64 standard normal,
input drawn first then filter) and the FLOP formula (:70-74).  Operand
generation stays on the host with numpy so that GPU outputs can be compared
bit for bit against the reference's own outputs on identical inputs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .plan import GemmDims, TilePlan
from .tensors import ConvParams, output_dims
from .layouts import footprint_elems

BYTES_PER_ELEM = 4


@dataclass(frozen=True)
class BenchConfig:
    name: str
    c_in: int
    h_in: int
    w_in: int
    c_out: int
    h_f: int
    w_f: int
    stride: int
    batch: int = 2
    repeats: int = 10
    algorithm: str = "im2win-opt"
    plan: TilePlan | None = None
    seed: int = 0

    @property
    def params(self) -> ConvParams:
        return ConvParams(c_in=self.c_in, c_out=self.c_out, h_f=self.h_f, w_f=self.w_f,
                          stride=self.stride)

    @property
    def out_dims(self) -> tuple[int, int]:
        return output_dims(self.h_in, self.w_in, self.params)

    @property
    def flops(self) -> int:
        h_out, w_out = self.out_dims
        return 2 * self.batch * self.c_out * h_out * w_out * self.c_in * self.h_f * self.w_f

    def gemm_dims(self) -> GemmDims:
        h_out, w_out = self.out_dims
        return GemmDims(self.c_out, self.batch * h_out * w_out, self.c_in * self.h_f * self.w_f)

    @property
    def w_eff(self) -> int:
        h_out, w_out = self.out_dims
        return (w_out - 1) * self.stride + self.w_f

    def elems(self, layout: str) -> int:
        return footprint_elems(layout, self.batch, self.c_in, self.h_in, self.w_in, self.params)

    @property
    def out_elems(self) -> int:
        h_out, w_out = self.out_dims
        return self.batch * self.c_out * h_out * w_out

    @property
    def filter_elems(self) -> int:
        return self.c_out * self.c_in * self.h_f * self.w_f

    def transform_bytes(self) -> int:
        """Algorithmic HBM bytes of the transform: read the input once, write Ĩ once."""
        return BYTES_PER_ELEM * (self.elems("raw") + self.elems("im2win"))

    def conv_bytes(self, operand_bytes: int = 4) -> int:
        """Algorithmic HBM bytes of the convolution: read Ĩ and F once, write O once."""
        return operand_bytes * (self.elems("im2win") + self.filter_elems) + BYTES_PER_ELEM * self.out_elems

    def conv_nchw_bytes(self) -> int:
        """Algorithmic HBM bytes of the convolution that gathers its windows straight from the
        input (no Ĩ): read X and F once, write O once."""
        return BYTES_PER_ELEM * (self.elems("raw") + self.filter_elems + self.out_elems)


def _cfg(name, c_in, h_in, w_in, c_out, h_f, w_f, stride) -> BenchConfig:
    return BenchConfig(name=name, c_in=c_in, h_in=h_in, w_in=w_in, c_out=c_out, h_f=h_f,
                       w_f=w_f, stride=stride)


BENCHMARKS = {
    cfg.name: cfg
    for cfg in (
        _cfg("conv1", 3, 227, 227, 96, 11, 11, 4),
        _cfg("conv2", 3, 231, 231, 96, 11, 11, 4),
        _cfg("conv3", 3, 227, 227, 64, 7, 7, 2),
        _cfg("conv4", 64, 224, 224, 64, 7, 7, 2),
        _cfg("conv5", 96, 24, 24, 256, 5, 5, 1),
        _cfg("conv6", 256, 12, 12, 512, 3, 3, 1),
        _cfg("conv7", 3, 224, 224, 64, 3, 3, 1),
        _cfg("conv8", 64, 112, 112, 128, 3, 3, 1),
        _cfg("conv9", 64, 56, 56, 64, 3, 3, 1),
        _cfg("conv10", 128, 28, 28, 128, 3, 3, 1),
        _cfg("conv11", 256, 14, 14, 256, 3, 3, 1),
        _cfg("conv12", 512, 7, 7, 512, 3, 3, 1),
    )
}

# BASELINE.json configs[0]: N=8 C=64 56x56 K=64 3x3 s1 pad1, run as an explicit
# zero pad to 58x58 followed by the unpadded conv (the reference has no padding).
CONFIG1 = _cfg("cfg1-pad1", 64, 58, 58, 64, 3, 3, 1)
CONFIG1 = BenchConfig(**{**CONFIG1.__dict__, "batch": 8})


def make_inputs(cfg: BenchConfig) -> tuple[np.ndarray, np.ndarray]:
    """Seeded standard-normal input and filter (bench.py:152-159), host numpy float32."""
    rng = np.random.default_rng(cfg.seed)
    inp = rng.standard_normal((cfg.batch, cfg.c_in, cfg.h_in, cfg.w_in), dtype=np.float32)
    flt = rng.standard_normal((cfg.c_out, cfg.c_in, cfg.h_f, cfg.w_f), dtype=np.float32)
    return inp, flt


def make_config1_inputs(seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Config 1 operands: N(0,1) input 8x64x56x56 zero-padded to 58x58, filter 64x64x3x3."""
    rng = np.random.default_rng(seed)
    inp = rng.standard_normal((8, 64, 56, 56), dtype=np.float32)
    flt = rng.standard_normal((64, 64, 3, 3), dtype=np.float32)
    padded = np.zeros((8, 64, 58, 58), dtype=np.float32)
    padded[:, :, 1:57, 1:57] = inp
    return padded, flt
