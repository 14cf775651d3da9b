"""GPU parity: libstr (sm_100a) vs the fp64 oracle after every batch.

Tolerances (BASELINE.json north_star): relative Frobenius error of every core, and of the
fit, <= 1e-9 in the FP64 contraction mode and <= 1e-4 in the 3xTF32 mode."""
import numpy as np
import pytest

from tests._parity import gpu_stream

TOL = {"f64": 1e-9, "3xtf32": 1e-4}


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["T3", "T4", "T5", "P1"])
def test_parity_f64_small(name):
    for b, errs, fo, fg, h, orc in gpu_stream(name, contract="f64"):
        assert max(errs) <= TOL["f64"], (b, errs)
        assert abs(fg - fo) <= TOL["f64"] * fo, (b, fo, fg)


@pytest.mark.gpu
@pytest.mark.parametrize("name,contract", [("P2", "f64"), ("P3", "f64"), ("P5", "f64"), ("P6", "f64"), ("P2", "3xtf32"),
                                           ("P5", "3xtf32"), ("P6", "3xtf32")])
def test_parity_multi_tile(name, contract):
    """Sizes spanning several 64/128-row tiles with ragged tails, unequal ranks; P6 has
    R_nR_{n+1} up to 120 (the inverse's largest tile grids) and rank 12."""
    for b, errs, fo, fg, h, orc in gpu_stream(name, contract=contract):
        assert max(errs) <= TOL[contract], (b, errs)
        assert abs(fg - fo) <= TOL[contract] * fo, (b, fo, fg)


@pytest.mark.gpu
def test_parity_C1_every_batch():
    """configs[0] (C1, fp64) end to end: every batch, every core, fit."""
    for b, errs, fo, fg, h, orc in gpu_stream("C1", contract="f64"):
        assert max(errs) <= TOL["f64"], (b, errs)
        assert abs(fg - fo) <= TOL["f64"] * fo, (b, fo, fg)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 2])
def test_parity_split_points_agree(k):
    """Both two-pass split points k give the oracle's result (N=5)."""
    for b, errs, fo, fg, h, orc in gpu_stream("T5", contract="f64", split_k=k):
        assert max(errs) <= TOL["f64"], (b, errs)
