"""Relative error ||X - TR(G)||_F / ||X||_F (§4).

Test infrastructure only (see oracle/__init__.py).  X̂ is formed through
X̂_[N] = G_N(2) (G^{≠N}_[2])^T (Eq. tr_als P:160-164 with n = N) and the residual is taken
directly (never via ||X||^2 - 2<X,X̂> + ||X̂||^2).  Columns are processed in blocks that
share the last chain index i_{N-1} purely to bound memory.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np

from .tensor import unfold
from .tralg import core_unfold, subchain, unfold2


def residual_sums(X: np.ndarray, cores: Sequence[np.ndarray]):
    """(sum (X - X̂)^2, sum X^2) for X of shape (I_1..I_{N-1}, T) and temporal core with T rows."""
    N = X.ndim
    X = np.asarray(X, dtype=np.float64)
    XN = unfold(X, N, "mode")                          # T x prod I
    GN2 = core_unfold(cores[-1])                        # T x R_N R_1
    I_last = cores[N - 2].shape[1]
    blk = XN.shape[1] // I_last
    r2 = 0.0
    for i in range(I_last):
        S = unfold2(subchain(cores, N, last_index=i))  # blk x R_N R_1
        D = XN[:, i * blk:(i + 1) * blk] - GN2 @ S.T
        r2 += float(np.sum(D * D))
    return r2, float(np.sum(XN * XN))


def relative_error(X: np.ndarray, cores: Sequence[np.ndarray]) -> float:
    r2, x2 = residual_sums(X, cores)
    if x2 == 0.0:
        raise ValueError("relative error undefined for a zero tensor")
    return float(np.sqrt(r2 / x2))
