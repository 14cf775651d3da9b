"""Tensor substrate: linearization, Def. 1 unfoldings, TR format by definition.

Test infrastructure only (see oracle/__init__.py).  Indices are 0-based; mode numbers n are
1-based as in the paper.  A tensor X of order N is a numpy array of shape (I_1, ..., I_N)
indexed X[i_1, ..., i_N].
"""
from __future__ import annotations

import itertools
from typing import Sequence

import numpy as np


def linear_index(idx: Sequence[int], dims: Sequence[int]) -> int:
    """overline(i_1 ... i_N) = sum_n i_n prod_{j<n} I_j (P:119, 0-based)."""
    out, stride = 0, 1
    for n, (i, d) in enumerate(zip(idx, dims)):
        if not 0 <= i < d:
            raise ValueError(f"index {i} out of range for mode {n + 1} (size {d})")
        out += i * stride
        stride *= d
    return out


def unfold(X: np.ndarray, n: int, kind: str) -> np.ndarray:
    """Def. 1, element by element through linear_index.

    kind = 'classical' : X_(n)(i_n, overline(i_1..i_{n-1} i_{n+1}..i_N))
           'mode'      : X_[n](i_n, overline(i_{n+1}..i_N i_1..i_{n-1}))
           'prefix'    : X_<n>(overline(i_1..i_n), overline(i_{n+1}..i_N))
    The element-wise loop is used for small tensors; larger ones use the equivalent
    axis permutation + first-index-fastest reshape (checked against the loop in tests).
    """
    N = X.ndim
    if not 1 <= n <= N:
        raise ValueError(f"mode {n} invalid for an order-{N} tensor")
    dims = X.shape
    k = n - 1
    if kind == "classical":
        order = [k] + [j for j in range(N) if j != k]
        return np.transpose(X, order).reshape(dims[k], -1, order="F")
    if kind == "mode":
        order = [k] + list(range(k + 1, N)) + list(range(0, k))
        return np.transpose(X, order).reshape(dims[k], -1, order="F")
    if kind == "prefix":
        return X.reshape(int(np.prod(dims[:n])), -1, order="F")
    raise ValueError(kind)


def unfold_loop(X: np.ndarray, n: int, kind: str) -> np.ndarray:
    """Def. 1 written as the literal element-wise assignment (tiny tensors only)."""
    N, dims, k = X.ndim, X.shape, n - 1
    if kind == "prefix":
        out = np.zeros((int(np.prod(dims[:n])), int(np.prod(dims[n:]))), X.dtype)
    else:
        out = np.zeros((dims[k], int(np.prod(dims)) // dims[k]), X.dtype)
    for idx in itertools.product(*[range(d) for d in dims]):
        if kind == "classical":
            cols = [j for j in range(N) if j != k]
            out[idx[k], linear_index([idx[j] for j in cols], [dims[j] for j in cols])] = X[idx]
        elif kind == "mode":
            cols = list(range(k + 1, N)) + list(range(0, k))
            out[idx[k], linear_index([idx[j] for j in cols], [dims[j] for j in cols])] = X[idx]
        else:
            out[linear_index(idx[:n], dims[:n]), linear_index(idx[n:], dims[n:])] = X[idx]
    return out


def fold(M: np.ndarray, n: int, kind: str, shape: Sequence[int]) -> np.ndarray:
    """Inverse of unfold (so fold(unfold(X)) == X exactly)."""
    N = len(shape)
    k = n - 1
    if kind == "prefix":
        return M.reshape(shape, order="F")
    if kind == "classical":
        order = [k] + [j for j in range(N) if j != k]
    elif kind == "mode":
        order = [k] + list(range(k + 1, N)) + list(range(0, k))
    else:
        raise ValueError(kind)
    permuted_shape = [shape[j] for j in order]
    Y = M.reshape(permuted_shape, order="F")
    return np.transpose(Y, np.argsort(order))


def tr_entry(cores: Sequence[np.ndarray], idx: Sequence[int]) -> float:
    """X(i_1..i_N) = Tr(G_1(i_1) G_2(i_2) ... G_N(i_N)), G_n(i) = G_n[:, i, :]."""
    prod = np.eye(cores[0].shape[0])
    for G, i in zip(cores, idx):
        prod = prod @ G[:, i, :]
    return float(np.trace(prod))


def tr_full_bruteforce(cores: Sequence[np.ndarray]) -> np.ndarray:
    """Whole TR tensor entry by entry from the trace definition (tiny shapes only)."""
    dims = [G.shape[1] for G in cores]
    X = np.zeros(dims)
    for idx in itertools.product(*[range(d) for d in dims]):
        X[idx] = tr_entry(cores, idx)
    return X


def frobenius(X: np.ndarray) -> float:
    return float(np.sqrt(np.sum(np.asarray(X, dtype=np.float64) ** 2)))
