"""rSTR-K: randomized streaming TR with the Kronecker sub-sampled randomized Fourier transform
(KSRFT, Def. 10; Alg. 5; update rules P:629-641; Alg. 9
P:1194-1258), step by step.

Test infrastructure only (see oracle/__init__.py).  Readings (R17-R22):
  R17 F_j is the unitary DFT, F_j(a, b) = exp(-2 pi i a b / I_j) / sqrt(I_j).
  R18 sign flips D_j come from the SplitMix64 stream of reading R11 with k = 0 (a slot the
      index draws never use): per step tau one stream of sum_j I_j draws, mode j's entries at
      offsets sum_{l<j} I_l .. (I_N = t_init at tau = 0, t_new afterwards); d = +1 when the top bit
      of the draw is 0, else -1.  Redrawn every step (Alg. 9 l.21 P:1224).
  R19 the sampled mixed slices (G^_k)_S are always taken from G_k mixed with the CURRENT step's
      D_k (Alg. 9 l.22-23 re-mix the cores every step; X^new is mixed with the same D), at the
      index table idxs(:,k) drawn when G_k last changed.
  R20 garbles of ledger #19: P_n <- P_n^old + X^_S conj(G^_S) (the extra "+P_n" of P:635 dropped);
      Q_n <- Q_n + G^_S^T conj(G^_S) with the conjugate of Alg. 9 l.1250 (P:637 omits it; without it
      Re(Q) is not the Gram of the real-constrained problem); the unhatted X, G of P:1249-1250 and
      the "init" superscripts of P:1232, P:1248 read as the hatted, new-data quantities; the init
      stage uses the same conjugated forms.
  R21 only Re(P_n), Re(Q_n) are ever read (Alg. 9 l.1251), so the state keeps the real
      parts: Re(A conj B) = Re A Re B + Im A Im B.
  R22 the temporal solve is the literal G_N^new = Re(X~_S[N]) (Re(G^_S[2]^T))^dagger (P:632,
      Alg. 9 l.1233), evaluated with an SVD pseudo-inverse (as reading R4).
Index draws are uniform with replacement (S in Def. 10) with the rSTR-U streams (R11).
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence

import numpy as np

from .rstream import sampled_fibers, sampled_subchain
from .sampler import MASK, draw_uniform, splitmix64, stream_key
from .tralg import core_fold, solve_right, symmetrize, unfold2


def dft_unitary(I: int) -> np.ndarray:
    """F (I x I): F(a, b) = exp(-2 pi i a b / I) / sqrt(I) (Def. 10; reading R17)."""
    a = np.arange(I)
    return np.exp(-2j * np.pi * np.outer(a, a) / I) / np.sqrt(I)


def sign_flips(seed: int, tau: int, N: int, dims: Sequence[int]) -> List[np.ndarray]:
    """D_1..D_N diagonals in {+1, -1} for step tau (Def. 10; reading R18)."""
    total = int(sum(dims))
    u, _ = splitmix64(stream_key(seed, tau, 0, N) & MASK, total)
    out, off = [], 0
    for I in dims:
        out.append(np.array([-1.0 if (x >> 63) else 1.0 for x in u[off:off + I]]))
        off += I
    return out


def mixing_matrices(signs: Sequence[np.ndarray]) -> List[np.ndarray]:
    """W_j = F_j D_j (Def. 10)."""
    return [dft_unitary(len(d)) * d[None, :] for d in signs]


def mode_product(X: np.ndarray, W: np.ndarray, j: int) -> np.ndarray:
    """X x_j W (mode-j product, 0-based j): Y(.., a, ..) = sum_i W(a, i) X(.., i, ..)."""
    Y = np.tensordot(W, X, axes=([1], [j]))       # new axis first
    return np.moveaxis(Y, 0, j)


def mix_tensor(X: np.ndarray, Ws: Sequence[np.ndarray]) -> np.ndarray:
    """X^ = X x_1 (F_1 D_1) x_2 ... x_N (F_N D_N) (Alg. 5 l.3 P:651; Alg. 9 l.4, l.22)."""
    Y = np.asarray(X, dtype=np.complex128)
    for j, W in enumerate(Ws):
        Y = mode_product(Y, W, j)
    return Y


def mix_core(G: np.ndarray, W: np.ndarray) -> np.ndarray:
    """G^ = G x_2 (F D) (Alg. 5 l.2 P:650; Alg. 9 l.3, l.23)."""
    return mode_product(np.asarray(G, dtype=np.complex128), W, 1)


def unmix_fibers(XS: np.ndarray, W: np.ndarray) -> np.ndarray:
    """X~_S[n] = D_n F_n^* X^_S[n] (Alg. 5 l.8 P:658; Alg. 9 l.1232, l.1248): W^H = D F^*."""
    return W.conj().T @ XS


class KSRFTStreamingTR:
    def __init__(self, X_init: np.ndarray, init_cores: Sequence[np.ndarray], m: int, seed: int,
                 draw_hook: Optional[Callable] = None):
        """Initialization stage of Alg. 9."""
        self.N = N = len(init_cores)
        self.m, self.seed, self.hook = m, seed, draw_hook
        self.cores: List[np.ndarray] = [np.array(G, dtype=np.float64) for G in init_cores]
        X_init = np.asarray(X_init, dtype=np.float64)
        for n in range(1, N + 1):
            G = self.cores[n - 1]
            if m < G.shape[0] * G.shape[2]:
                raise ValueError("rSTR requires m >= R_n R_{n+1} (SPEC S:451)")
        self.tau = 0
        self.idxs = np.zeros((m, N), dtype=np.int64)
        self.draws = {}
        self.signs = {}
        # l.2-4: D_j, F_j; mix cores and the init tensor
        self.W = self._mixers(X_init.shape)
        Xh = mix_tensor(X_init, self.W)
        # l.5-8: idxs(:,k), (G^_k)_S
        for k in range(1, N + 1):
            self._draw(k, X_init.shape[k - 1])
        self.P: List[np.ndarray] = []
        self.Q: List[np.ndarray] = []
        for n in range(1, N):                               # l.9-20 (reading R20, R21)
            GS2 = unfold2(sampled_subchain(self._sampled(), N, n))
            XS = unmix_fibers(sampled_fibers(Xh, self.idxs, n), self.W[n - 1])
            self.P.append(np.real(XS @ GS2.conj()))
            self.Q.append(symmetrize(np.real(GS2.T @ GS2.conj())))
        self.t_processed = X_init.shape[-1]

    def _mixers(self, shape) -> List[np.ndarray]:
        d = sign_flips(self.seed, self.tau, self.N, shape)
        self.signs[self.tau] = d
        return mixing_matrices(d)

    def _sampled(self) -> List[np.ndarray]:
        """(G^_k)_S = (G_k x_2 W_k)(:, idxs(:,k), :) with the current W_k (reading R19).  The
        temporal core contributes only its rows of the current step (G_N^new)."""
        out = []
        for k in range(1, self.N + 1):
            G = self.cores[k - 1]
            if k == self.N:
                if self.tN != self.W[k - 1].shape[0]:   # last step's rows: not on the temporal chain
                    out.append(None)
                    continue
                G = G[:, G.shape[1] - self.tN:, :]
            out.append(mix_core(G, self.W[k - 1])[:, self.idxs[:, k - 1], :])
        return out

    def _draw(self, k: int, I: int) -> None:
        """idxs(:,k) <- Randsample(I_k, m) (uniform with replacement, Def. 10)."""
        if self.hook is not None:
            ind = np.asarray(self.hook(self.tau, k, I, None), dtype=np.int64)
        else:
            ind = draw_uniform(self.seed, self.tau, k, self.N, I, self.m)
        self.draws[(self.tau, k)] = ind.copy()
        self.idxs[:, k - 1] = ind
        if k == self.N:
            self.tN = I

    def update(self, X_new: np.ndarray) -> None:
        """One time step, Alg. 9 l.21-56."""
        N = self.N
        X_new = np.asarray(X_new, dtype=np.float64)
        self.tau += 1
        tn = X_new.shape[-1]
        # l.22-24: redefine D_j, mix X^new and the cores (R18, R19)
        self.W = self._mixers(X_new.shape)
        Xh = mix_tensor(X_new, self.W)
        # temporal mode, l.26-34: chain of (G^_k)_S, k = 1..N-1
        samp = self._sampled()
        GS2 = unfold2(sampled_subchain(samp, N, N))                         # m x R_N R_1 (complex)
        XS = unmix_fibers(sampled_fibers(Xh, self.idxs, N), self.W[N - 1])  # t_new x m
        GN_new2 = np.real(XS) @ np.linalg.pinv(np.real(GS2.T), rcond=1e-12)  # reading R22
        RN, R1 = self.cores[-1].shape[0], self.cores[-1].shape[2]
        self.cores[-1] = np.concatenate([self.cores[-1], core_fold(GN_new2, RN, R1)], axis=1)
        # l.35-37: G^_N^new, idxs(:,N) over [t_new], (G^_N^new)_S
        self._draw(N, tn)
        for n in range(1, N):                                                # l.39-55
            GS2 = unfold2(sampled_subchain(self._sampled(), N, n))          # m x R_nR_{n+1}
            XS = unmix_fibers(sampled_fibers(Xh, self.idxs, n), self.W[n - 1])
            self.P[n - 1] = self.P[n - 1] + np.real(XS @ GS2.conj())        # R20, R21
            self.Q[n - 1] = symmetrize(self.Q[n - 1] + np.real(GS2.T @ GS2.conj()))
            G = self.cores[n - 1]
            self.cores[n - 1] = core_fold(solve_right(self.P[n - 1], self.Q[n - 1]), G.shape[0], G.shape[2])
            self._draw(n, G.shape[1])                                        # l.53-54
        self.t_processed += tn
