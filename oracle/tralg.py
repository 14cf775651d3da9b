"""TR algebra (§2): subchains, products, Gram tensors, Gram chains, solves.

Test infrastructure only (see oracle/__init__.py).  Cores are numpy arrays in the paper's
layout G_n of shape (R_n, I_n, R_{n+1}); the lateral slice is G_n(i) = G_n[:, i, :].
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np

from .tensor import fold, unfold


# ----------------------------------------------------------------------------- products
def subchain_product(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Mode-2 subchain product A ⊠₂ B (Def. 6).

    A: I_1 x J_1 x K, B: K x J_2 x I_2 -> I_1 x J_1J_2 x I_2 with
    (A ⊠₂ B)(overline(j_1 j_2)) = A(j_1) B(j_2)   (j_1 fastest).
    """
    I1, J1, K = A.shape
    K2, J2, I2 = B.shape
    assert K == K2
    C = np.einsum("ajk,kml->amjl", A, B)          # [a, j2, j1, l]
    return C.reshape(I1, J1 * J2, I2)               # index j2*J1 + j1 = overline(j1 j2)


def slices_hadamard(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Mode-2 slices-Hadamard product A ⊡₂ B (Def. 7): (A ⊡₂ B)(j) = A(j) B(j)."""
    assert A.shape[1] == B.shape[1] and A.shape[2] == B.shape[0]
    return np.einsum("ajk,kjl->ajl", A, B)


def outer(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Outer product (Def. 4)."""
    return np.multiply.outer(A, B)


def contract_2413(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """General contracted product A ×_{2,4}^{1,3} B (Def. 5).

    A: I_1 x J x R_1 x K, B: J x I_2 x K x R_2 ->
    (i_1, i_2, r_1, r_2) = sum_{j,k} A(i_1, j, r_1, k) B(j, i_2, k, r_2).
    """
    return np.einsum("ajrk,jbks->abrs", A, B)


# ----------------------------------------------------------------------------- subchains
def subchain_order(N: int, n: int) -> List[int]:
    """Core order of G^{≠n}: n+1, ..., N, 1, ..., n-1 (Def. 3; Eq. P:296)."""
    return list(range(n + 1, N + 1)) + list(range(1, n))


def subchain(cores: Sequence[np.ndarray], n: int, last_index: Optional[int] = None) -> np.ndarray:
    """Subchain tensor G^{≠n} (Def. 3) of shape R_{n+1} x prod_{j≠n} I_j x R_n,

    built as G_{n+1} ⊠₂ ... ⊠₂ G_N ⊠₂ G_1 ⊠₂ ... ⊠₂ G_{n-1} (Eq. P:294-297).
    With ``last_index`` = i the last core of the chain is restricted to its slice i, giving
    the contiguous block of rows whose last chain index equals i (used only to bound memory
    in the matrix product X_[n] G^{≠n}_[2], which is then summed block by block).
    """
    N = len(cores)
    order = subchain_order(N, n)
    T = cores[order[0] - 1]
    if len(order) == 1 and last_index is not None:
        T = T[:, last_index:last_index + 1, :]
    for pos, j in enumerate(order[1:], start=1):
        G = cores[j - 1]
        if last_index is not None and pos == len(order) - 1:
            G = G[:, last_index:last_index + 1, :]
        T = subchain_product(T, G)
    return T


def unfold2(T3: np.ndarray) -> np.ndarray:
    """Mode-2 unfolding [2] of a 3rd-order tensor (Def. 1): (j, overline(r_3 r_1))."""
    return unfold(T3, 2, "mode")


def core_unfold(G: np.ndarray) -> np.ndarray:
    """G_n(2): classical mode-2 unfolding, I_n x R_nR_{n+1}, column r_n + R_n r_{n+1}."""
    return unfold(G, 2, "classical")


def core_fold(M: np.ndarray, Rn: int, Rn1: int) -> np.ndarray:
    """Reshape G_n(2) back to the core tensor G_n (R_n x I_n x R_{n+1})."""
    return fold(M, 2, "classical", (Rn, M.shape[0], Rn1))


# ----------------------------------------------------------------------------- Grams
def gram_core(G: np.ndarray) -> np.ndarray:
    """Z_n = sum_i G_n(i)^T ∘ G_n(i)^T (Alg. 2 l.2 P:228; Alg. 4 l.2 P:362).

    Z(a, b, c, d) = sum_i G(b, i, a) G(d, i, c); shape R_{n+1} x R_n x R_{n+1} x R_n.
    """
    Z = np.zeros((G.shape[2], G.shape[0], G.shape[2], G.shape[0]))
    for i in range(G.shape[1]):
        S = G[:, i, :].T
        Z += outer(S, S)
    return Z


def gram_chain(Zs: Sequence[np.ndarray]) -> np.ndarray:
    """Z_a ×_{2,4}^{1,3} Z_b ×_{2,4}^{1,3} ... evaluated left to right (Alg. 2 l.5 P:231)."""
    H = Zs[0]
    for Z in Zs[1:]:
        H = contract_2413(H, Z)
    return H


def chain_order(N: int, n: int) -> List[int]:
    """Gram-chain order for H^{≠n}: n-1, ..., 1, N, ..., n+1 (Alg. 4 l.5 P:365)."""
    return list(range(n - 1, 0, -1)) + list(range(N, n, -1))


def gram_unfold(H: np.ndarray) -> np.ndarray:
    """H_<2>: rows overline(i_1 i_2), columns overline(r_1 r_2) (Def. 1)."""
    return unfold(H, 2, "prefix")


# ----------------------------------------------------------------------------- solves
def pinv_sym(Q: np.ndarray, rcond: float = 1e-12) -> np.ndarray:
    """Q^† for symmetric PSD Q: eigen-decomposition, eigenvalues below
    rcond * lambda_max dropped (reading R3)."""
    Qs = 0.5 * (Q + Q.T)
    w, V = np.linalg.eigh(Qs)
    lam_max = w.max() if w.size else 0.0
    inv = np.zeros_like(w)
    keep = w > rcond * lam_max
    inv[keep] = 1.0 / w[keep]
    return (V * inv) @ V.T


def solve_right(P: np.ndarray, Q: np.ndarray, refine: int = 2) -> np.ndarray:
    """G = P Q^† (Alg. 4 l.9, l.17) with Q^† of pinv_sym (reading R3), evaluated to
    full fp64 accuracy: G_0 = P Q^†, then ``refine`` steps of iterative refinement
    G_{k+1} = G_k + (P - G_k Q) Q^† with the residual formed in extended precision (np.longdouble).
    The plain product P Q^† carries an error of order cond(Q)·eps — about 1e-9 relative at the
    cond(Q) ~ 1e7 that C3 reaches from its TR-ALS init, the size of the fp64 parity bar itself —
    while the refined solution is accurate to about eps_ld·cond(Q) (eps_ld = 2^-64: ~1e-12 at
    cond 1e7; tests/test_oracle_tralg.py pins it against exact and 60-digit solutions).  P's rows lie in the
    range of Q (P = X G^{≠n}, Q = G^{≠n T} G^{≠n}), so the corrections stay in it and a
    rank-deficient Q still gets the minimum-norm solution."""
    Qs = symmetrize(Q)
    Qp = pinv_sym(Qs)
    G = P @ Qp
    if refine:
        Ql = Qs.astype(np.longdouble)
        Pl = np.asarray(P, dtype=np.longdouble)
        for _ in range(refine):
            R = (Pl - G.astype(np.longdouble) @ Ql).astype(np.float64)
            G = G + R @ Qp
    return G


def symmetrize(Q: np.ndarray) -> np.ndarray:
    """(Q + Q^T)/2 after every accumulation (reading R5)."""
    return 0.5 * (Q + Q.T)
