"""Oracle pins: TR format, subchains, Grams, Prop. 1, pseudo-inverse (§2).

Mandated self-checks 1 (TR brute force) and 2 (Gram via core Grams)."""
import itertools

import numpy as np
import pytest

from oracle.tensor import fold, tr_full_bruteforce, unfold
from oracle.tralg import (chain_order, core_fold, core_unfold, gram_chain, gram_core, gram_unfold, pinv_sym, solve_right,
                          slices_hadamard, subchain, subchain_order, subchain_product, unfold2)

CASES = [((3, 4, 2), (2, 3, 4)), ((3, 2, 4, 2), (2, 3, 4, 2)), ((2, 3, 2, 2, 3), (2, 3, 2, 4, 3))]


def _cores(dims, ranks, seed=0):
    rng = np.random.default_rng(seed)
    N = len(dims)
    return [rng.standard_normal((ranks[n], dims[n], ranks[(n + 1) % N])) for n in range(N)]


@pytest.mark.parametrize("dims,ranks", CASES)
def test_tr_bruteforce_equals_unfolding_product(dims, ranks):
    """Self-check 1: Tr(G_1(i_1)...G_N(i_N)) == fold(G_n(2) G^{≠n}_[2]^T) (Eq. P:160-164) for every n."""
    cores = _cores(dims, ranks)
    X = tr_full_bruteforce(cores)
    for n in range(1, len(dims) + 1):
        Xn = core_unfold(cores[n - 1]) @ unfold2(subchain(cores, n)).T
        rel = np.linalg.norm(fold(Xn, n, "mode", dims) - X) / np.linalg.norm(X)
        assert rel < 1e-13


@pytest.mark.parametrize("dims,ranks", CASES)
def test_subchain_slices_match_definition(dims, ranks):
    """Def. 3: slice overline(i_{n+1}..i_N i_1..i_{n-1}) = prod of the slices."""
    cores = _cores(dims, ranks, 1)
    N = len(dims)
    for n in range(1, N + 1):
        S = subchain(cores, n)
        order = subchain_order(N, n)
        for idx in itertools.islice(itertools.product(*[range(dims[j - 1]) for j in order]), 0, None, 3):
            prod = np.eye(ranks[n % N])
            for j, i in zip(order, idx):
                prod = prod @ cores[j - 1][:, i, :]
            lin = sum(i * int(np.prod([dims[j - 1] for j in order[:p]])) for p, i in enumerate(idx))
            np.testing.assert_allclose(S[:, lin, :], prod, rtol=1e-13, atol=1e-13)


def test_subchain_order2_special_case():
    cores = _cores((3, 4), (2, 3), 2)
    np.testing.assert_array_equal(subchain(cores, 1), cores[1])
    np.testing.assert_array_equal(subchain(cores, 2), cores[0])


def test_subchain_blocks_concatenate():
    cores = _cores((3, 2, 4, 2), (2, 3, 4, 2), 3)
    for n in range(1, 5):
        full = subchain(cores, n)
        last = (n - 1) if n > 1 else 4
        blocks = [subchain(cores, n, last_index=i) for i in range(cores[last - 1].shape[1])]
        np.testing.assert_allclose(np.concatenate(blocks, axis=1), full, rtol=0, atol=0)


def test_products_small_cases():
    rng = np.random.default_rng(4)
    A = rng.standard_normal((2, 3, 4))
    B = rng.standard_normal((4, 5, 3))
    C = subchain_product(A, B)
    for j1, j2 in itertools.product(range(3), range(5)):
        np.testing.assert_allclose(C[:, j1 + 3 * j2, :], A[:, j1, :] @ B[:, j2, :], rtol=1e-14)
    D = rng.standard_normal((4, 3, 2))
    H = slices_hadamard(A, D)
    for j in range(3):
        np.testing.assert_allclose(H[:, j, :], A[:, j, :] @ D[:, j, :], rtol=1e-14)


def test_gram_core_is_index_swapped_core_gram():
    """Z(a,b,c,d) = sum_i G(b,i,a) G(d,i,c) equals (G_(2)^T G_(2))[b + R_n a, d + R_n c]."""
    rng = np.random.default_rng(5)
    G = rng.standard_normal((3, 7, 4))
    Z = gram_core(G)
    M = core_unfold(G).T @ core_unfold(G)
    Rn = 3
    for a, b, c, d in itertools.product(range(4), range(3), range(4), range(3)):
        assert abs(Z[a, b, c, d] - M[b + Rn * a, d + Rn * c]) < 1e-12


@pytest.mark.parametrize("dims,ranks", CASES)
def test_prop1_gram_chain_equals_explicit_gram(dims, ranks):
    """Self-check 2: (Z_{n-1} × ... × Z_1 × Z_N × ... × Z_{n+1})_<2> == G^{≠n}_[2]^T G^{≠n}_[2]
    (Prop. 1; Alg. 4 l.5 P:365), also with a new temporal block in place of G_N."""
    cores = _cores(dims, ranks, 6)
    N = len(dims)
    Z = [gram_core(G) for G in cores]
    for n in range(1, N + 1):
        S2 = unfold2(subchain(cores, n))
        H = gram_unfold(gram_chain([Z[j - 1] for j in chain_order(N, n)]))
        np.testing.assert_allclose(H, S2.T @ S2, rtol=1e-12, atol=1e-12 * np.abs(H).max())
    GN_new = np.random.default_rng(7).standard_normal((ranks[-1], 3, ranks[0]))
    ZN_new = gram_core(GN_new)
    cores_new = cores[:-1] + [GN_new]
    for n in range(1, N):
        S2 = unfold2(subchain(cores_new, n))
        H = gram_unfold(gram_chain([ZN_new if j == N else Z[j - 1] for j in chain_order(N, n)]))
        np.testing.assert_allclose(H, S2.T @ S2, rtol=1e-12, atol=1e-12 * np.abs(H).max())


def test_core_fold_roundtrip():
    G = np.random.default_rng(8).standard_normal((3, 5, 2))
    np.testing.assert_array_equal(core_fold(core_unfold(G), 3, 2), G)
    # column r_n + R_n r_{n+1}
    M = core_unfold(G)
    assert M[4, 2 + 3 * 1] == G[2, 4, 1]


def test_pinv_sym():
    rng = np.random.default_rng(9)
    A = rng.standard_normal((20, 6))
    Q = A.T @ A
    np.testing.assert_allclose(pinv_sym(Q), np.linalg.inv(Q), rtol=1e-10)
    B = rng.standard_normal((6, 3))
    Qd = B @ B.T                         # rank 3 PSD
    Pd = pinv_sym(Qd)
    np.testing.assert_allclose(Qd @ Pd @ Qd, Qd, atol=1e-10)
    np.testing.assert_allclose(Pd @ Qd @ Pd, Pd, atol=1e-10)
    np.testing.assert_allclose(Pd, np.linalg.pinv(Qd, rcond=1e-10), atol=1e-10)


def _unimodular_spd(S, rng, spread=3):
    """Q = L L^T with L unit lower triangular with integer entries: an SPD integer matrix whose
    inverse L^{-T} L^{-1} is an integer matrix too (det L = 1), with a large condition number."""
    L = np.tril(rng.integers(-spread, spread + 1, (S, S)), -1) + np.eye(S, dtype=np.int64)
    return L @ L.T


@pytest.mark.parametrize("S,spread,seed", [(6, 3, 0), (12, 3, 1), (16, 2, 0), (20, 2, 1), (24, 1, 2)])
def test_solve_right_exact_on_unimodular_systems(S, spread, seed):
    """Closed form: with Q = L L^T (L unimodular, integer) and an integer G, P = G Q is exact in fp64
    and the solution of G Q = P is G itself.  The refined solve reaches it to a few ulps even where
    cond(Q) (1e6-2e7, the range C3 reaches) makes the plain P Q^† miss it by cond·eps ~ 1e-9."""
    rng = np.random.default_rng(seed)
    Q = _unimodular_spd(S, rng, spread)
    G = rng.integers(-5, 6, (4, S))
    P = G @ Q
    assert np.abs(P).max() < 2 ** 52 and np.abs(Q).max() < 2 ** 52
    Qf, Pf = Q.astype(np.float64), P.astype(np.float64)
    cond = np.linalg.cond(Qf)
    assert 1e6 < cond < 1e8
    err = np.linalg.norm(solve_right(Pf, Qf) - G) / np.linalg.norm(G)
    assert err < 1e-13, (S, cond, err)
    err0 = np.linalg.norm(solve_right(Pf, Qf, refine=0) - G) / np.linalg.norm(G)
    assert err0 > 100 * err


def test_solve_right_matches_mpmath_on_random_ill_conditioned():
    """Reference solution in 60-digit arithmetic (mpmath LU) for an SPD Q of cond 1e7."""
    import mpmath
    rng = np.random.default_rng(5)
    S = 10
    U, _ = np.linalg.qr(rng.standard_normal((S, S)))
    Q = (U * np.logspace(0, 7, S)) @ U.T
    Q = 0.5 * (Q + Q.T)
    P = rng.standard_normal((3, S)) @ Q + 1e-3 * rng.standard_normal((3, S))
    mpmath.mp.dps = 60
    Qm = mpmath.matrix(Q.tolist())
    ref = np.array([[float(v) for v in (mpmath.lu_solve(Qm, mpmath.matrix(P[i].tolist())))] for i in range(3)])
    err = np.linalg.norm(solve_right(P, Q) - ref) / np.linalg.norm(ref)
    assert err < 1e-13, err
    err0 = np.linalg.norm(solve_right(P, Q, refine=0) - ref) / np.linalg.norm(ref)
    assert err0 > 100 * err
