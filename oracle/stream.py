"""STR — streaming TR decomposition, Alg. 4, step by step.

Test infrastructure only (see oracle/__init__.py).  Every quantity is formed from its
plain definition in fp64:
  * subchains G^{≠n} are materialized by the ⊠₂ chain (Def. 3 / Eq. P:294-297),
  * X_[n] is the Def. 1 mode-n unfolding,
  * Q increments are Gram chains of the Z's (Prop. 1; Alg. 4 l.15),
  * G = P Q^† uses the symmetric pseudo-inverse (reading R3).
Readings of the paper: R1 Z_N is computed at init; R2 the full Z_N
of l.11 is recomputed but only Z_N^new enters the loop; R5 Q is symmetrized after each
accumulation.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np

from .tensor import unfold
from .tralg import (chain_order, core_fold, core_unfold, gram_chain, gram_core, gram_unfold,
                    solve_right, subchain, symmetrize, unfold2)

# Above this many subchain entries the product X_[n] G^{≠n}_[2] is summed over blocks of
# rows sharing the last chain index (memory bound only; same sum, block by block).
_BLOCK_ENTRIES = 2 ** 25


def mode_n_times_subchain(X: np.ndarray, cores: Sequence[np.ndarray], n: int) -> np.ndarray:
    """M_n = X_[n] G^{≠n}_[2]  (Alg. 4 l.4 P:364, l.9 P:370, l.14 P:376).

    X has shape (I_1, ..., I_N) with I_N the length of the temporal block whose core
    (cores[N-1]) enters the subchain.
    """
    N = len(cores)
    Xn = unfold(X, n, "mode")                              # I_n x J (columns cyclic)
    J = Xn.shape[1]
    Rn, Rn1 = cores[n - 1].shape[0], cores[n - 1].shape[2]
    if J * Rn * Rn1 <= _BLOCK_ENTRIES:
        return Xn @ unfold2(subchain(cores, n))
    last = (n - 1) if n > 1 else N                         # last core of the chain (1-based)
    I_last = cores[last - 1].shape[1]
    blk = J // I_last
    M = np.zeros((Xn.shape[0], Rn * Rn1))
    for i in range(I_last):                                # rows with last index i are contiguous
        M += Xn[:, i * blk:(i + 1) * blk] @ unfold2(subchain(cores, n, last_index=i))
    return M


class StreamingTR:
    """State and update of Alg. 4.  Cores in paper layout; G_N is R_N x T x R_1."""

    def __init__(self, X_init: np.ndarray, init_cores: Sequence[np.ndarray]):
        """Initialization stage, Alg. 4 l.1-5."""
        self.N = N = len(init_cores)
        self.cores: List[np.ndarray] = [np.array(G, dtype=np.float64) for G in init_cores]
        assert X_init.shape[:-1] == tuple(G.shape[1] for G in self.cores[:-1])
        assert X_init.shape[-1] == self.cores[-1].shape[1]
        X_init = np.asarray(X_init, dtype=np.float64)
        # l.2 Z_1..Z_{N-1}; Z_N as well because l.5's chain uses it (reading R1).
        self.Z = [gram_core(G) for G in self.cores]
        self.P: List[Optional[np.ndarray]] = [None] * (N - 1)
        self.Q: List[Optional[np.ndarray]] = [None] * (N - 1)
        for n in range(1, N):
            # l.4 P_n = X^init_[n] G^{≠n}_[2]
            self.P[n - 1] = mode_n_times_subchain(X_init, self.cores, n)
            # l.5 Q_n = (Z_{n-1} × ... × Z_1 × Z_N × ... × Z_{n+1})_<2>
            H = gram_chain([self.Z[j - 1] for j in chain_order(N, n)])
            self.Q[n - 1] = symmetrize(gram_unfold(H))
        self.t_processed = X_init.shape[-1]

    @classmethod
    def empty(cls, cores: Sequence[np.ndarray]) -> "StreamingTR":
        """State with no history: P_n = 0, Q_n = 0, zero temporal rows (used by the pin
        'one STR step from an empty history = one TR-ALS sweep')."""
        self = cls.__new__(cls)
        self.N = N = len(cores)
        self.cores = [np.array(G, dtype=np.float64) for G in cores[:-1]]
        RN, R1 = cores[-1].shape[0], cores[-1].shape[2]
        self.cores.append(np.zeros((RN, 0, R1)))
        self.Z = [gram_core(G) for G in self.cores]
        self.P = [np.zeros((self.cores[n].shape[1], self.cores[n].shape[0] * self.cores[n].shape[2]))
                  for n in range(N - 1)]
        self.Q = [np.zeros((p.shape[1], p.shape[1])) for p in self.P]
        self.t_processed = 0
        return self

    def update(self, X_new: np.ndarray) -> None:
        """One time step τ: Alg. 4 l.7-19."""
        N = self.N
        X_new = np.asarray(X_new, dtype=np.float64)
        cores = self.cores
        # ---- temporal mode
        # l.8 H^{≠N} = Z_{N-1} × ... × Z_1
        H_N = gram_chain([self.Z[j - 1] for j in chain_order(N, N)])
        # l.9 G_N(2)^new = X^new_[N] G^{≠N}_[2] (H^{≠N}_<2>)^†   (subchain uses old cores)
        M_N = mode_n_times_subchain(X_new, cores[:-1] + [cores[-1][:, :0, :]], N)
        GN_new2 = solve_right(M_N, symmetrize(gram_unfold(H_N)))
        RN, R1 = cores[-1].shape[0], cores[-1].shape[2]
        GN_new = core_fold(GN_new2, RN, R1)                                # R_N x t_new x R_1
        # l.10 append the new rows
        cores[-1] = np.concatenate([cores[-1], GN_new], axis=1)
        # l.11 Z_N over the whole temporal core (reading R2: computed, not used below)
        self.Z[N - 1] = gram_core(cores[-1])
        # Z_N^new: Gram of the new rows only
        Z_N_new = gram_core(GN_new)
        # ---- non-temporal modes, Gauss-Seidel order
        for n in range(1, N):
            # l.13 G^{≠n}_new with G_N^new in the temporal slot (Eq. partial2)
            cores_new = cores[:-1] + [GN_new]
            # l.14 P_n += X^new_[n] (G^{≠n}_new)_[2]
            self.P[n - 1] = self.P[n - 1] + mode_n_times_subchain(X_new, cores_new, n)
            # l.15 H^{≠n}_new = (×_{n-1..1} Z_j) × Z_N^new × (×_{N-1..n+1} Z_j)
            Zs = [Z_N_new if j == N else self.Z[j - 1] for j in chain_order(N, n)]
            H = gram_chain(Zs)
            # l.16 Q_n += (H^{≠n}_new)_<2>
            self.Q[n - 1] = symmetrize(self.Q[n - 1] + gram_unfold(H))
            # l.17 G_n(2) = P_n Q_n^†, reshape
            Rn, Rn1 = cores[n - 1].shape[0], cores[n - 1].shape[2]
            cores[n - 1] = core_fold(solve_right(self.P[n - 1], self.Q[n - 1]), Rn, Rn1)
            # l.18 Z_n refresh
            self.Z[n - 1] = gram_core(cores[n - 1])
        self.t_processed += X_new.shape[-1]
        self.last_GN_new = GN_new

    def state_scalars(self) -> int:
        """Stored scalars of {temporal core rows, P, Q, Z_1..Z_{N-1}} — the accounting of the
        memory formula (2(N-1)I + t_old)R^2 + (N-1)R^4 of P:705-707 without the
        I^{N-1}t_new batch and with the non-temporal cores counted in the (N-1)IR^2 term."""
        n = self.cores[-1].size
        n += sum(p.size for p in self.P) + sum(G.size for G in self.cores[:-1])
        n += sum(q.size for q in self.Q)
        return n
