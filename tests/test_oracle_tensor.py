"""Oracle pins: linearization and Def. 1 unfoldings."""
import os

import numpy as np
import pytest

from oracle.tensor import fold, linear_index, tr_entry, tr_full_bruteforce, unfold, unfold_loop

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_rows(name):
    rows = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            key, *vals = line.split()
            rows.setdefault(key, []).append([float(v) for v in vals])
    return {k: np.array(v) for k, v in rows.items()}


def test_linear_index_examples():
    # P:119 with 0-based indices: first index fastest; last element = prod(dims) - 1.
    assert linear_index((0, 0, 0), (2, 3, 4)) == 0
    assert linear_index((1, 0, 0), (2, 3, 4)) == 1
    assert linear_index((1, 2, 3), (2, 3, 4)) == 23
    with pytest.raises(ValueError):
        linear_index((0, 3, 0), (2, 3, 4))


def test_unfold_worked_example():
    X = np.arange(1, 9, dtype=float).reshape((2, 2, 2), order="F")
    g = _golden_rows("unfold_2x2x2.txt")
    np.testing.assert_array_equal(unfold(X, 2, "classical"), g["classical2"])
    np.testing.assert_array_equal(unfold(X, 2, "mode"), g["mode2"])
    np.testing.assert_array_equal(unfold(X, 1, "prefix"), g["prefix1"])


@pytest.mark.parametrize("shape", [(2, 3, 4), (3, 2, 2, 3), (2, 3, 2, 2, 2)])
def test_unfold_matches_elementwise_definition(shape):
    rng = np.random.default_rng(1)
    X = rng.standard_normal(shape)
    for n in range(1, len(shape) + 1):
        for kind in ("classical", "mode", "prefix"):
            U = unfold(X, n, kind)
            np.testing.assert_array_equal(U, unfold_loop(X, n, kind))
            np.testing.assert_array_equal(fold(U, n, kind, shape), X)


def test_mode_and_classical_same_columns():
    # Π_n is a column permutation: same multiset of columns.
    rng = np.random.default_rng(2)
    X = rng.standard_normal((3, 4, 2, 5))
    for n in range(1, 5):
        A = unfold(X, n, "classical")
        B = unfold(X, n, "mode")
        assert sorted(map(tuple, A.T.round(12))) == sorted(map(tuple, B.T.round(12)))


def test_trace_definition_special_cases():
    # rank-1 cores: X = product of scalars; identity slices: X == R everywhere.
    rng = np.random.default_rng(3)
    cores = [rng.standard_normal((1, d, 1)) for d in (2, 3, 2)]
    X = tr_full_bruteforce(cores)
    ref = np.einsum("i,j,k->ijk", cores[0][0, :, 0], cores[1][0, :, 0], cores[2][0, :, 0])
    np.testing.assert_allclose(X, ref, rtol=1e-14)
    R = 3
    eye = [np.repeat(np.eye(R)[:, None, :], d, axis=1) for d in (2, 2, 3)]
    np.testing.assert_array_equal(tr_full_bruteforce(eye), np.full((2, 2, 3), float(R)))
    assert tr_entry(eye, (1, 0, 2)) == R
