"""TR-ALS, Alg. 1 — init producer and pin for one STR step.

Test infrastructure only (see oracle/__init__.py).  Each mode update solves the LS problem
of Eq. (tr_als), min || G^{≠n}_[2] G_n(2)^T - X_[n]^T ||_F, with LAPACK lstsq on the
explicitly materialized subchain (no normal equations, no Gram chains) so that it is an
independent route to the same LS solutions STR forms through Prop. 1.
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np

from .fit import relative_error
from .tensor import unfold
from .tralg import core_fold, subchain, unfold2


def als_mode_update(X: np.ndarray, cores: List[np.ndarray], n: int) -> None:
    """Alg. 1 l.4-5 for one mode n (1-based), in place."""
    A = unfold2(subchain(cores, n))                  # J x R_nR_{n+1}
    B = unfold(X, n, "mode").T                       # J x I_n
    sol = np.linalg.lstsq(A, B, rcond=None)[0]       # R_nR_{n+1} x I_n
    G = cores[n - 1]
    cores[n - 1] = core_fold(sol.T, G.shape[0], G.shape[2])


def tr_als_sweep(X: np.ndarray, cores: Sequence[np.ndarray], order: Sequence[int]) -> List[np.ndarray]:
    """One sweep of Alg. 1 l.3-6 over the given mode order; returns new cores."""
    out = [np.array(G, dtype=np.float64) for G in cores]
    for n in order:
        als_mode_update(X, out, n)
    return out


def tr_als(X: np.ndarray, ranks: Sequence[int], init: Sequence[np.ndarray], tol: float = 1e-8,
           max_sweeps: int = 100):
    """Alg. 1 with the §4 termination rule: stop when the change in relative error
    between two sweeps is below ``tol`` or after ``max_sweeps`` sweeps (reading R20)."""
    N = X.ndim
    cores = [np.array(G, dtype=np.float64) for G in init]
    prev = relative_error(X, cores)
    sweeps = 0
    for sweeps in range(1, max_sweeps + 1):
        cores = tr_als_sweep(X, cores, range(1, N + 1))
        err = relative_error(X, cores)
        if abs(prev - err) < tol:
            break
        prev = err
    return cores, err, sweeps
