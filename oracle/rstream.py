"""rSTR-U / rSTR-L: Alg. 7 and Alg. 8, step by step.

Test infrastructure only (see oracle/__init__.py).  Readings: R4 the temporal
solve X_S ((G_S[2])^T)^† is evaluated literally with an SVD pseudo-inverse; R6 draws are with
replacement; R7 X(idxs(:,1), ..., :, ..., idxs(:,N)) is the *zipped* fiber selection (column s
uses row s of idxs); R8 no rescaling D_n; R9 Alg. 8 samples G_N^new after the temporal solve;
R10 leverage rank threshold 1e-12; R11 SplitMix64 draws keyed by (seed, tau, k).

``draw_hook(tau, k, I, p)`` may replace the sampler (returns m indices); the GPU parity
tests use it to replay the index tables the library reports, and the degeneracy pin uses it
to inject the full Cartesian enumeration.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence

import numpy as np

from .sampler import draw_uniform, draw_weighted, leverage_distribution
from .tralg import core_fold, core_unfold, slices_hadamard, solve_right, subchain_order, symmetrize, unfold2


def sampled_subchain(sampled: Sequence[np.ndarray], N: int, n: int) -> np.ndarray:
    """G^{≠n}_S: start from identity lateral slices (R_{n+1} x m x R_{n+1}) and apply
    ⊡₂ with (G_k)_S for k = n+1..N, 1..n-1 (Alg. 3 l.5-7 P:268-271; Alg. 7)."""
    order = subchain_order(N, n)
    first = sampled[order[0] - 1]
    R, m = first.shape[0], first.shape[1]
    T = np.repeat(np.eye(R)[:, None, :], m, axis=1)
    for k in order:
        T = slices_hadamard(T, sampled[k - 1])
    return T


def sampled_fibers(X: np.ndarray, idxs: np.ndarray, n: int) -> np.ndarray:
    """X_S[n]: I_n x m, column s = X(idxs[s,0], ..., :, ..., idxs[s,N-1]) (reading R7)."""
    N = X.ndim
    cols = []
    for s in range(idxs.shape[0]):
        key = tuple(slice(None) if j == n - 1 else int(idxs[s, j]) for j in range(N))
        cols.append(X[key])
    return np.stack(cols, axis=1)


class RandomizedStreamingTR:
    def __init__(self, X_init: np.ndarray, init_cores: Sequence[np.ndarray], m: int, kind: str,
                 seed: int, draw_hook: Optional[Callable] = None):
        """Initialization stage of Alg. 7 / Alg. 8."""
        assert kind in ("uniform", "leverage")
        self.N = N = len(init_cores)
        self.m, self.kind, self.seed, self.hook = m, kind, seed, draw_hook
        self.cores: List[np.ndarray] = [np.array(G, dtype=np.float64) for G in init_cores]
        X_init = np.asarray(X_init, dtype=np.float64)
        for n in range(1, N):
            if m < self.cores[n - 1].shape[0] * self.cores[n - 1].shape[2]:
                raise ValueError("rSTR requires m >= R_n R_{n+1} (SPEC S:451)")
        self.tau = 0
        self.idxs = np.zeros((m, N), dtype=np.int64)
        self.sampled: List[Optional[np.ndarray]] = [None] * N
        self.draws = {}                     # (tau, k) -> indices, for replay / inspection
        for k in range(1, N + 1):           # Alg. 7 l.2-5 / Alg. 8 l.2-6
            self._draw(k, self.cores[k - 1])
        self.P: List[np.ndarray] = []
        self.Q: List[np.ndarray] = []
        for n in range(1, N):               # Alg. 7 l.6-16
            GS2 = unfold2(sampled_subchain(self.sampled, N, n))
            XS = sampled_fibers(X_init, self.idxs, n)
            self.P.append(XS @ GS2)
            self.Q.append(symmetrize(GS2.T @ GS2))
        self.t_processed = X_init.shape[-1]

    def _draw(self, k: int, G: np.ndarray) -> None:
        """idxs(:,k) <- Randsample(I_k, m[, true, p_k]); (G_k)_S <- G_k(:, idxs(:,k), :)."""
        I = G.shape[1]
        p = leverage_distribution(core_unfold(G)) if self.kind == "leverage" else None
        if self.hook is not None:
            ind = np.asarray(self.hook(self.tau, k, I, p), dtype=np.int64)
        elif self.kind == "uniform":
            ind = draw_uniform(self.seed, self.tau, k, self.N, I, self.m)
        else:
            ind = draw_weighted(self.seed, self.tau, k, self.N, p, self.m)
        self.draws[(self.tau, k)] = ind.copy()
        self.idxs[:, k - 1] = ind
        self.sampled[k - 1] = G[:, ind, :]

    def update(self, X_new: np.ndarray) -> None:
        """One time step, Alg. 7 l.17-41 / Alg. 8 l.18-43."""
        N = self.N
        X_new = np.asarray(X_new, dtype=np.float64)
        self.tau += 1
        # temporal: G^{≠N}_S from the cached samples of G_1..G_{N-1}
        GS2 = unfold2(sampled_subchain(self.sampled, N, N))                 # m x R_N R_1
        XS = sampled_fibers(X_new, self.idxs, N)                             # t_new x m
        GN_new2 = XS @ np.linalg.pinv(GS2.T, rcond=1e-12)                    # reading R4
        RN, R1 = self.cores[-1].shape[0], self.cores[-1].shape[2]
        GN_new = core_fold(GN_new2, RN, R1)
        self.cores[-1] = np.concatenate([self.cores[-1], GN_new], axis=1)
        # idxs(:,N) over [t_new]; (G_N^new)_S  (reading R9 for Alg. 8)
        self._draw(N, GN_new)
        for n in range(1, N):
            GS2 = unfold2(sampled_subchain(self.sampled, N, n))              # m x R_nR_{n+1}
            XS = sampled_fibers(X_new, self.idxs, n)                         # I_n x m
            self.P[n - 1] = self.P[n - 1] + XS @ GS2
            self.Q[n - 1] = symmetrize(self.Q[n - 1] + GS2.T @ GS2)
            G = self.cores[n - 1]
            self.cores[n - 1] = core_fold(solve_right(self.P[n - 1], self.Q[n - 1]), G.shape[0], G.shape[2])
            self._draw(n, self.cores[n - 1])
        self.t_processed += X_new.shape[-1]
