"""Oracle pins for rSTR (Alg. 7 / Alg. 8), the sampler and leverage scores."""
import itertools
import os

import numpy as np
import pytest

from oracle.rstream import RandomizedStreamingTR
from oracle.sampler import (draw_uniform, draw_weighted, leverage_distribution, leverage_scores, splitmix64,
                            stream_key)
from oracle.stream import StreamingTR
from oracle.tralg import core_unfold, subchain, unfold2
from workloads import make_stream
from workloads.gen import paper_view

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_reference_vector():
    with open(os.path.join(GOLDEN, "splitmix64.txt")) as f:
        vals = dict(line.split() for line in f if line.strip() and not line.startswith("#"))
    out, _ = splitmix64(0, 1)
    assert out[0] == int(vals["state0_first"], 16)


def test_uniform_frequencies():
    """Uniform Randsample with replacement: empirical frequencies within ±0.02."""
    idx = draw_uniform(seed=5, tau=0, k=1, N=3, I=4, m=40000)
    assert idx.min() >= 0 and idx.max() <= 3
    freq = np.bincount(idx, minlength=4) / idx.size
    assert np.all(np.abs(freq - 0.25) < 0.02)


def test_weighted_frequencies_and_support():
    p = np.array([0.5, 0.0, 0.3, 0.2])
    idx = draw_weighted(seed=9, tau=2, k=3, N=4, p=p, m=40000)
    freq = np.bincount(idx, minlength=4) / idx.size
    assert freq[1] == 0.0
    assert np.all(np.abs(freq - p) < 0.02)


def test_stream_keys_distinct():
    keys = {stream_key(7, tau, k, 5) for tau in range(20) for k in range(1, 6)}
    assert len(keys) == 100


def test_leverage_scores_qr_svd_and_sum():
    """Def. 8: ℓ_i = ||Q(i,:)||^2 for any orthonormal basis Q — QR and SVD agree; Σℓ = rank."""
    rng = np.random.default_rng(1)
    A = rng.standard_normal((50, 7))
    ell, r = leverage_scores(A)
    Qm, _ = np.linalg.qr(A)
    np.testing.assert_allclose(ell, np.sum(Qm * Qm, axis=1), rtol=1e-12, atol=1e-14)
    assert r == 7 and abs(ell.sum() - 7) < 1e-12
    B = rng.standard_normal((50, 3)) @ rng.standard_normal((3, 7))      # rank 3
    ell, r = leverage_scores(B)
    assert r == 3 and abs(ell.sum() - 3) < 1e-10
    # I <= R^2 with full row rank: all scores 1, p uniform (reading R10)
    C = rng.standard_normal((6, 9))
    np.testing.assert_allclose(leverage_distribution(C), np.full(6, 1 / 6), rtol=1e-12)


def test_lemma1_product_distribution_bound():
    """Lemma 1: q^{≠n}(i) = prod_{m≠n} p_m(i_m) >= beta_n p^{≠n}(i), brute force."""
    rng = np.random.default_rng(2)
    dims, ranks = (6, 5, 7), (2, 2, 3)
    N = 3
    cores = [rng.standard_normal((ranks[n], dims[n], ranks[(n + 1) % N])) for n in range(N)]
    p = [leverage_distribution(core_unfold(G)) for G in cores]
    for n in range(1, N + 1):
        S2 = unfold2(subchain(cores, n))
        ell, r = leverage_scores(S2)
        pn = ell / r
        order = list(range(n + 1, N + 1)) + list(range(1, n))
        beta = 1.0 / (ranks[n - 1] * ranks[n % N] *
                      np.prod([ranks[m - 1] ** 2 for m in range(1, N + 1) if m not in (n, n % N + 1)]))
        for lin, idx in enumerate(itertools.product(*[range(dims[j - 1]) for j in reversed(order)])):
            idx = tuple(reversed(idx))                     # first chain index fastest
            q = np.prod([p[j - 1][i] for j, i in zip(order, idx)])
            assert q >= beta * pn[lin] - 1e-15


@pytest.mark.parametrize("kind", ["uniform", "leverage"])
def test_rstr_exhaustive_enumeration_equals_str(kind):
    """rSTR ≡ STR when every draw injects the full Cartesian table over (i_1..i_{N-1}, t)
    (SURVEY.md Appendix A.12): t_init = t_new so m is constant."""
    cfg = make_stream("T4").cfg.with_(t_init=3, t_new=3)
    s = make_stream(cfg)
    N = cfg.N
    full = np.array(list(itertools.product(*[range(d) for d in reversed(cfg.dims + (cfg.t_new,))])))[:, ::-1]
    m = full.shape[0]

    def hook(tau, k, I, p):
        return full[:, k - 1]

    Xi = paper_view(s.init_slab()).astype(np.float64)
    r = RandomizedStreamingTR(Xi, s.init_cores(), m, kind, seed=1, draw_hook=hook)
    d = StreamingTR(Xi, s.init_cores())
    for b in range(3):
        Xb = paper_view(s.batch(b)).astype(np.float64)
        r.update(Xb)
        d.update(Xb)
        for n in range(N):
            rel = np.linalg.norm(r.cores[n] - d.cores[n]) / np.linalg.norm(d.cores[n])
            assert rel < 1e-10, (b, n, rel)


@pytest.mark.parametrize("kind", ["uniform", "leverage"])
def test_rstr_deterministic_and_Q_psd(kind):
    cfg = make_stream("T4").cfg
    s = make_stream(cfg)
    runs = []
    for _ in range(2):
        r = RandomizedStreamingTR(paper_view(s.init_slab()), s.init_cores(), 40, kind, seed=3)
        for b in range(2):
            before = [q.copy() for q in r.Q]
            r.update(paper_view(s.batch(b)))
            for q0, q1 in zip(before, r.Q):
                assert np.linalg.eigvalsh(q1 - q0).min() > -1e-10 * np.trace(q1)
        runs.append(r)
    for a, b in zip(runs[0].cores, runs[1].cores):
        np.testing.assert_array_equal(a, b)
    assert runs[0].draws.keys() == runs[1].draws.keys()


def test_rstr_requires_enough_rows():
    s = make_stream("T4")
    with pytest.raises(ValueError):
        RandomizedStreamingTR(paper_view(s.init_slab()), s.init_cores(), 5, "uniform", seed=1)


def test_uniform_sketch_is_unbiased():
    """Monte-Carlo pin of the sampled normal equations (Alg. 7 l.15-16 with uniform rows drawn with
    replacement, no rescaling, reading R8): over the seeded draws, E[X_S G_S] = (m/J) X_[n] G^{≠n}_[2]
    and E[G_S^T G_S] = (m/J) G^{≠n T} G^{≠n} with J = prod_{j≠n} I_j, the exact products built by
    the independent ⊠₂ subchain route."""
    from oracle.rstream import sampled_fibers, sampled_subchain
    from oracle.tensor import unfold
    rng = np.random.default_rng(21)
    dims, ranks = (4, 3, 5), (2, 3, 2)
    N, m, n = 3, 6, 2
    cores = [rng.standard_normal((ranks[k], dims[k], ranks[(k + 1) % N])) for k in range(N)]
    X = rng.standard_normal(dims)
    J = int(np.prod([d for k, d in enumerate(dims) if k != n - 1]))
    Gsub = unfold2(subchain(cores, n))
    P_ref = (m / J) * unfold(X, n, "mode") @ Gsub
    Q_ref = (m / J) * Gsub.T @ Gsub
    P_sum = np.zeros_like(P_ref)
    Q_sum = np.zeros_like(Q_ref)
    trials = 3000
    for s in range(trials):
        idxs = np.stack([draw_uniform(1000 + s, 0, k, N, dims[k - 1], m) for k in range(1, N + 1)], axis=1)
        samp = [G[:, idxs[:, k], :] for k, G in enumerate(cores)]
        GS2 = unfold2(sampled_subchain(samp, N, n))
        P_sum += sampled_fibers(X, idxs, n) @ GS2
        Q_sum += GS2.T @ GS2
    # the mean of `trials` i.i.d. sketches: relative error ~ 1/sqrt(trials m) ~ 0.8%
    assert np.linalg.norm(P_sum / trials - P_ref) / np.linalg.norm(P_ref) < 0.05
    assert np.linalg.norm(Q_sum / trials - Q_ref) / np.linalg.norm(Q_ref) < 0.05


def test_leverage_sketch_expectation():
    """Monte-Carlo pin of Alg. 8's sampled normal equations (rows drawn with replacement from the
    product of the per-mode leverage distributions p_k = l(G_k(2))/rank, Lemma 1; no rescaling,
    reading R8): E[X_S G_S] = m X_[n] diag(q) G^{≠n}_[2] and E[G_S^T G_S] = m G^{≠n T} diag(q) G^{≠n},
    q(i) = prod_{j≠n} p_j(i_j) over the subchain rows (first chain index fastest), brute force."""
    from oracle.rstream import sampled_fibers, sampled_subchain
    from oracle.tensor import unfold
    rng = np.random.default_rng(23)
    dims, ranks = (7, 6, 8), (1, 2, 1)          # I_k > R_k R_{k+1}: non-uniform leverage scores
    N, m, n = 3, 5, 1
    cores = [rng.standard_normal((ranks[k], dims[k], ranks[(k + 1) % N])) * rng.uniform(0.2, 3.0, (1, dims[k], 1))
             for k in range(N)]
    X = rng.standard_normal(dims)
    p = [leverage_distribution(core_unfold(G)) for G in cores]
    assert max(np.max(pk) * len(pk) for pk in p) > 1.3        # genuinely non-uniform
    order = list(range(n + 1, N + 1)) + list(range(1, n))
    q = np.array([np.prod([p[j - 1][i] for j, i in zip(order, tuple(reversed(idx)))])
                  for idx in itertools.product(*[range(dims[j - 1]) for j in reversed(order)])])
    Gsub = unfold2(subchain(cores, n))
    P_ref = m * unfold(X, n, "mode") @ (q[:, None] * Gsub)
    Q_ref = m * Gsub.T @ (q[:, None] * Gsub)
    P_sum = np.zeros_like(P_ref)
    Q_sum = np.zeros_like(Q_ref)
    trials = 3000
    for s in range(trials):
        idxs = np.stack([draw_weighted(3000 + s, 0, k, N, p[k - 1], m) for k in range(1, N + 1)], axis=1)
        samp = [G[:, idxs[:, k], :] for k, G in enumerate(cores)]
        GS2 = unfold2(sampled_subchain(samp, N, n))
        P_sum += sampled_fibers(X, idxs, n) @ GS2
        Q_sum += GS2.T @ GS2
    assert np.linalg.norm(P_sum / trials - P_ref) / np.linalg.norm(P_ref) < 0.06
    assert np.linalg.norm(Q_sum / trials - Q_ref) / np.linalg.norm(Q_ref) < 0.06
