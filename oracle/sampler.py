"""Index draws for rSTR (Alg. 3 l.2-4 P:264-266; Alg. 7 P:1090, P:1113, P:1128;
Alg. 8) and leverage distributions (Def. 8 P:544-552,
Lemma 1).

Test infrastructure only (see oracle/__init__.py).  The paper leaves the RNG unspecified;
DESIGN.md reading R11 fixes a counter-based SplitMix64 generator that the CUDA library
re-implements independently (bit-identical uniform draws by construction):

  stream key   s0 = seed XOR (0x9E3779B97F4A7C15 * (1 + tau*(N+1) + k))   mod 2^64
               (tau = 0 for the init draws, tau = 1, 2, ... for update steps; k = mode 1..N)
  next()       s += 0x9E3779B97F4A7C15; z = s;
               z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9; z = (z ^ (z >> 27)) * 0x94D049BB133111EB;
               return z ^ (z >> 31)
  uniform      index = (u64 * I) >> 64                     (with replacement)
  weighted     c = left-to-right fp64 cumulative sum of p; target = (u64 >> 11) * 2^-53 * c[I-1];
               index = first i with c[i] > target, clamped to I-1
"""
from __future__ import annotations

from typing import Optional

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
MASK = (1 << 64) - 1


def stream_key(seed: int, tau: int, k: int, N: int) -> int:
    return (seed ^ ((GOLDEN * (1 + tau * (N + 1) + k)) & MASK)) & MASK


def splitmix64(state: int, count: int):
    """Return (list of count outputs, new state)."""
    out = []
    s = state
    for _ in range(count):
        s = (s + GOLDEN) & MASK
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        out.append(z ^ (z >> 31))
    return out, s


def draw_uniform(seed: int, tau: int, k: int, N: int, I: int, m: int) -> np.ndarray:
    """Randsample(I, m) with replacement, uniform on [I] (Alg. 7)."""
    u, _ = splitmix64(stream_key(seed, tau, k, N), m)
    return np.array([(x * I) >> 64 for x in u], dtype=np.int64)


def draw_weighted(seed: int, tau: int, k: int, N: int, p: np.ndarray, m: int) -> np.ndarray:
    """Randsample(I, m, true, p) (Alg. 3 l.3; Alg. 8): inverse-CDF draw with replacement."""
    p = np.asarray(p, dtype=np.float64)
    c = np.empty_like(p)
    acc = 0.0
    for i, v in enumerate(p):          # left-to-right fp64 cumulative sum
        acc = acc + float(v)
        c[i] = acc
    u, _ = splitmix64(stream_key(seed, tau, k, N), m)
    out = np.empty(m, dtype=np.int64)
    total = c[-1]
    for s, x in enumerate(u):
        target = float(x >> 11) * (2.0 ** -53) * total
        idx = int(np.searchsorted(c, target, side="right"))   # first i with c[i] > target
        out[s] = min(idx, len(p) - 1)
    return out


def leverage_scores(A: np.ndarray, rcond: float = 1e-12):
    """ℓ_i(A) = ||U(i,:)||^2, U an orthonormal basis of range(A) (Def. 8).

    U is taken from the thin SVD, keeping singular directions with sigma^2 > rcond*sigma_max^2
    (the numerical rank of reading R10).  Returns (scores, rank).
    """
    U, s, _ = np.linalg.svd(np.asarray(A, dtype=np.float64), full_matrices=False)
    if s.size == 0 or s[0] == 0.0:
        return np.zeros(A.shape[0]), 0
    keep = s ** 2 > rcond * s[0] ** 2
    Uk = U[:, keep]
    return np.sum(Uk * Uk, axis=1), int(keep.sum())


def leverage_distribution(G2: np.ndarray) -> np.ndarray:
    """p_n(i) = ℓ_i(G_n(2)) / rank(G_n(2)) (Lemma 1)."""
    ell, r = leverage_scores(G2)
    return ell / r
