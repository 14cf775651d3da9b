"""Oracle pins for rSTR-K (KSRFT, Def. 10; Alg. 5; Alg. 9).

Each pin checks the oracle against something other than itself: numpy's FFT, brute-force sums
over every index, the unitarity that makes an exhaustive KSRFT sketch exact (so the sketched
normal equations must equal the deterministic oracle's X_[n] G^{≠n}_[2] and G^{≠n T} G^{≠n}, built
by the independent ⊠₂ subchain route), and the exact-stream fixed point."""
import itertools

import numpy as np
import pytest

from oracle.ksrft import (KSRFTStreamingTR, dft_unitary, mix_core, mix_tensor, mixing_matrices, sign_flips,
                          unmix_fibers)
from oracle.rstream import sampled_fibers, sampled_subchain
from oracle.sampler import draw_uniform, splitmix64, stream_key
from oracle.stream import StreamingTR
from oracle.tensor import tr_full_bruteforce, unfold
from oracle.tralg import subchain, unfold2
from workloads import make_stream
from workloads.gen import paper_view


@pytest.mark.parametrize("I", [1, 2, 5, 8, 12])
def test_dft_is_numpy_ortho_fft_and_unitary(I):
    F = dft_unitary(I)
    np.testing.assert_allclose(F, np.fft.fft(np.eye(I), axis=0, norm="ortho"), atol=1e-14)
    np.testing.assert_allclose(F @ F.conj().T, np.eye(I), atol=1e-13)


def test_sign_flips_values_frequency_and_stream():
    d = sign_flips(seed=11, tau=3, N=4, dims=(4000, 3000, 2000, 1000))
    allv = np.concatenate(d)
    assert set(np.unique(allv)) <= {-1.0, 1.0}
    assert abs(allv.mean()) < 0.03
    # stream k = 0 of reading R11, top bit -> sign; consecutive draws across modes
    u, _ = splitmix64(stream_key(11, 3, 0, 4), 4001)
    assert d[1][0] == (-1.0 if u[4000] >> 63 else 1.0)
    # distinct from every index stream (k = 1..N)
    idx_keys = {stream_key(11, t, k, 4) for t in range(10) for k in range(1, 5)}
    assert stream_key(11, 3, 0, 4) not in idx_keys
    # fresh signs every step (Alg. 9 l.21)
    d2 = sign_flips(seed=11, tau=4, N=4, dims=(4000, 3000, 2000, 1000))
    assert np.mean(d2[0] != d[0]) > 0.4


def _tiny_cores(rng, dims, ranks):
    N = len(dims)
    return [rng.standard_normal((ranks[n], dims[n], ranks[(n + 1) % N])) for n in range(N)]


def test_mix_tensor_bruteforce():
    """X^(a) = sum_i prod_j W_j(a_j, i_j) X(i), every index enumerated (Alg. 5 l.3)."""
    rng = np.random.default_rng(3)
    dims = (3, 4, 2)
    X = rng.standard_normal(dims)
    Ws = mixing_matrices(sign_flips(5, 1, 3, dims))
    Y = mix_tensor(X, Ws)
    ref = np.zeros(dims, dtype=complex)
    for a in itertools.product(*[range(d) for d in dims]):
        for i in itertools.product(*[range(d) for d in dims]):
            ref[a] += Ws[0][a[0], i[0]] * Ws[1][a[1], i[1]] * Ws[2][a[2], i[2]] * X[i]
    np.testing.assert_allclose(Y, ref, atol=1e-12)


def test_mixed_tr_is_tr_of_mixed_cores():
    """TR(G_1..G_N) x_j (F_j D_j) for all j = TR(G^_1..G^_N) (multilinearity, Alg. 5 l.2-3)."""
    rng = np.random.default_rng(4)
    dims, ranks = (3, 4, 5), (2, 3, 2)
    cores = _tiny_cores(rng, dims, ranks)
    Ws = mixing_matrices(sign_flips(6, 2, 3, dims))
    Xh = mix_tensor(tr_full_bruteforce(cores), Ws)
    mixed = [mix_core(G, W) for G, W in zip(cores, Ws)]
    ref = np.zeros(dims, dtype=complex)
    for idx in itertools.product(*[range(d) for d in dims]):
        P = np.eye(ranks[0], dtype=complex)
        for G, i in zip(mixed, idx):
            P = P @ G[:, i, :]
        ref[idx] = np.trace(P)
    np.testing.assert_allclose(Xh, ref, atol=1e-12)


def test_unmixed_fibers_are_the_partial_mix_bruteforce():
    """D_n F_n^* applied to fibers of X^ = X mixed on every mode but n (Alg. 5 l.8)."""
    rng = np.random.default_rng(5)
    dims = (3, 4, 2)
    X = rng.standard_normal(dims)
    Ws = mixing_matrices(sign_flips(8, 1, 3, dims))
    idxs = np.stack([rng.integers(0, d, 7) for d in dims], axis=1)
    for n in (1, 2, 3):
        XS = unmix_fibers(sampled_fibers(mix_tensor(X, Ws), idxs, n), Ws[n - 1])
        for s in range(7):
            for i_n in range(dims[n - 1]):
                acc = 0.0
                for i in itertools.product(*[range(d) for d in dims]):
                    if i[n - 1] != i_n:
                        continue
                    w = 1.0
                    for j in range(3):
                        if j != n - 1:
                            w = w * Ws[j][idxs[s, j], i[j]]
                    acc += w * X[i]
                assert abs(XS[i_n, s] - acc) < 1e-12


def test_exhaustive_sketch_is_exact_normal_equations():
    """With idxs = the full Cartesian table, sum_s conj(W(s,i)) W(s,i') = delta (unitary mixing), so
    Re(X~_S conj G^_S) = X_[n] G^{≠n}_[2] and Re(G^_S^T conj G^_S) = G^{≠n T} G^{≠n} (the
    deterministic oracle's quantities via ⊠₂ subchains).  Fails on a dropped conjugate, on X and
    cores mixed with different signs, or on a wrong unmix."""
    rng = np.random.default_rng(6)
    dims, ranks = (3, 4, 2), (2, 3, 2)
    N = 3
    cores = _tiny_cores(rng, dims, ranks)
    X = rng.standard_normal(dims)
    Ws = mixing_matrices(sign_flips(9, 1, N, dims))
    full = np.array(list(itertools.product(*[range(d) for d in reversed(dims)])))[:, ::-1]
    Xh = mix_tensor(X, Ws)
    samp = [mix_core(G, W)[:, full[:, k], :] for k, (G, W) in enumerate(zip(cores, Ws))]
    for n in range(1, N + 1):
        GS2 = unfold2(sampled_subchain(samp, N, n))
        XS = unmix_fibers(sampled_fibers(Xh, full, n), Ws[n - 1])
        # every (i_{≠n}) combination appears I_n times in the full table (once per i_n value)
        P = np.real(XS @ GS2.conj()) / dims[n - 1]
        Q = np.real(GS2.T @ GS2.conj()) / dims[n - 1]
        Gsub = unfold2(subchain(cores, n))
        np.testing.assert_allclose(P, unfold(X, n, "mode") @ Gsub, atol=1e-11)
        np.testing.assert_allclose(Q, Gsub.T @ Gsub, atol=1e-11)


def test_exact_stream_fixed_point():
    """Noise-free exact TR stream from the true cores: every sketched LS problem is consistent,
    so rSTR-K keeps the true cores (Alg. 9 on exact data; reading R22's Re-LS included)."""
    rng = np.random.default_rng(7)
    dims, ranks, t0, tn = (5, 6, 4), (2, 3, 2, 2), 4, 3
    N = 4
    cores = _tiny_cores(rng, dims + (t0 + 2 * tn,), ranks)
    X = tr_full_bruteforce(cores)
    init = [G.copy() for G in cores[:-1]] + [cores[-1][:, :t0, :].copy()]
    r = KSRFTStreamingTR(X[..., :t0], init, m=40, seed=3)
    for b in range(2):
        r.update(X[..., t0 + b * tn:t0 + (b + 1) * tn])
    for n in range(N):
        rel = np.linalg.norm(r.cores[n] - cores[n]) / np.linalg.norm(cores[n])
        assert rel < 1e-10, (n, rel)


def test_rstrk_tracks_str_and_is_deterministic():
    s = make_stream("R4")
    cfg = s.cfg
    runs = []
    for _ in range(2):
        r = KSRFTStreamingTR(paper_view(s.init_slab()), s.init_cores(), cfg.sketch_rows, seed=7)
        for b in range(2):
            before = [q.copy() for q in r.Q]
            r.update(paper_view(s.batch(b)))
            for q0, q1 in zip(before, r.Q):   # each increment is a Gram: PSD
                assert np.linalg.eigvalsh(q1 - q0).min() > -1e-10 * np.trace(q1)
        runs.append(r)
    for a, b in zip(runs[0].cores, runs[1].cores):
        np.testing.assert_array_equal(a, b)
    d = StreamingTR(paper_view(s.init_slab()), s.init_cores())
    for b in range(2):
        d.update(paper_view(s.batch(b)))
    for n in range(cfg.N):   # a sketch of the same LS problems: close to STR, not equal
        rel = np.linalg.norm(runs[0].cores[n] - d.cores[n]) / np.linalg.norm(d.cores[n])
        assert 1e-6 < rel < 5e-2, (n, rel)
    # uniform index streams of rSTR-U (reading R11)
    np.testing.assert_array_equal(runs[0].draws[(1, 2)], draw_uniform(7, 1, 2, cfg.N, cfg.dims[1], cfg.sketch_rows))


def test_m_below_rank_product_rejected():
    s = make_stream("R4")
    with pytest.raises(ValueError):
        KSRFTStreamingTR(paper_view(s.init_slab()), s.init_cores(), 3, seed=1)


def test_ksrft_sketch_is_unbiased():
    """Monte-Carlo pin: for fixed signs D, uniform rows of the unitary-mixed problem give
    E[Re(X~_S conj G^_S)] = (m/J) X_[n] G^{≠n}_[2] and E[Re(G^_S^T conj G^_S)] = (m/J) G^{≠n T} G^{≠n}
    (unitarity of ⊗ F_j D_j), checked against the ⊠₂ subchain route over seeded index draws."""
    rng = np.random.default_rng(22)
    dims, ranks = (4, 3, 5), (2, 3, 2)
    N, m, n = 3, 6, 1
    cores = _tiny_cores(rng, dims, ranks)
    X = rng.standard_normal(dims)
    Ws = mixing_matrices(sign_flips(5, 1, N, dims))
    Xh = mix_tensor(X, Ws)
    mixed = [mix_core(G, W) for G, W in zip(cores, Ws)]
    J = int(np.prod([d for k, d in enumerate(dims) if k != n - 1]))
    Gsub = unfold2(subchain(cores, n))
    P_ref = (m / J) * unfold(X, n, "mode") @ Gsub
    Q_ref = (m / J) * Gsub.T @ Gsub
    P_sum = np.zeros_like(P_ref)
    Q_sum = np.zeros_like(Q_ref)
    trials = 3000
    for s in range(trials):
        idxs = np.stack([draw_uniform(2000 + s, 0, k, N, dims[k - 1], m) for k in range(1, N + 1)], axis=1)
        samp = [G[:, idxs[:, k], :] for k, G in enumerate(mixed)]
        GS2 = unfold2(sampled_subchain(samp, N, n))
        XS = unmix_fibers(sampled_fibers(Xh, idxs, n), Ws[n - 1])
        P_sum += np.real(XS @ GS2.conj())
        Q_sum += np.real(GS2.T @ GS2.conj())
    assert np.linalg.norm(P_sum / trials - P_ref) / np.linalg.norm(P_ref) < 0.05
    assert np.linalg.norm(Q_sum / trials - Q_ref) / np.linalg.norm(Q_ref) < 0.05
