"""Oracle pins for STR (Alg. 4): temporal solve, empty-history identity, post-init identity,
exact-stream fixed point, invariants.  Mandated self-checks 3 and 4."""
import numpy as np
import pytest

import oracle.stream as ost
from oracle.als import als_mode_update, tr_als, tr_als_sweep
from oracle.fit import relative_error
from oracle.stream import StreamingTR, mode_n_times_subchain
from oracle.tensor import frobenius, tr_full_bruteforce, unfold
from oracle.tralg import core_unfold, subchain, unfold2
from workloads import make_stream
from workloads.gen import paper_view


def _cores(dims, ranks, seed=0, scale=1.0):
    rng = np.random.default_rng(seed)
    N = len(dims)
    return [scale * rng.standard_normal((ranks[n], dims[n], ranks[(n + 1) % N])) for n in range(N)]


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("cfg", ["T3", "T4", "T5"])
def test_temporal_solve_rows_are_lstsq(cfg):
    """Alg. 4 l.9: each new temporal row equals LAPACK lstsq(G^{≠N}_[2], X_t)."""
    s = make_stream(cfg)
    st = StreamingTR(paper_view(s.init_slab()), s.init_cores())
    old = [G.copy() for G in st.cores]
    Xb = paper_view(s.batch(0)).astype(np.float64)
    st.update(Xb)
    N = st.N
    A = unfold2(subchain(old, N))
    ref = np.linalg.lstsq(A, unfold(Xb, N, "mode").T, rcond=None)[0].T
    np.testing.assert_allclose(core_unfold(st.last_GN_new), ref, rtol=1e-9, atol=1e-11)


@pytest.mark.parametrize("dims,ranks", [((5, 4), (2, 3, 4)), ((4, 3, 5), (2, 3, 4, 2)),
                                        ((3, 4, 3, 2), (2, 3, 2, 4, 3))])
def test_empty_history_step_equals_als_sweep(dims, ranks):
    """Self-check 4: one STR step from an empty history (P = Q = 0, no temporal rows) on X equals
    one TR-ALS sweep (Alg. 1) in mode order N, 1, ..., N-1 from the same cores, every core."""
    N = len(dims) + 1
    t = 6
    cores = _cores(dims + (t,), ranks, 11)
    X = np.random.default_rng(12).standard_normal(dims + (t,))
    st = StreamingTR.empty(cores)
    st.update(X)
    ref = tr_als_sweep(X, cores, [N] + list(range(1, N)))
    for n in range(N):
        assert _rel(st.cores[n], ref[n]) < 1e-10, n


@pytest.mark.parametrize("cfg", ["T3", "T4", "T5"])
def test_post_init_step_modes_N_and_1_equal_frozen_als(cfg):
    """After str_init, one STR step equals TR-ALS on [X_init; X_new] with the old temporal rows
    frozen for modes N and 1 exactly (Eq. partial); later modes use stale P."""
    s = make_stream(cfg)
    Xi = paper_view(s.init_slab()).astype(np.float64)
    Xb = paper_view(s.batch(0)).astype(np.float64)
    init = s.init_cores()
    st = StreamingTR(Xi, init)
    st.update(Xb)
    N = st.N
    Xcat = np.concatenate([Xi, Xb], axis=-1)
    # mode N (new rows only; old rows frozen): LS on X_new with old cores
    A = unfold2(subchain(init, N))
    ref_new = np.linalg.lstsq(A, unfold(Xb, N, "mode").T, rcond=None)[0].T
    np.testing.assert_allclose(core_unfold(st.cores[-1])[Xi.shape[-1]:], ref_new, rtol=1e-9, atol=1e-11)
    # mode 1: TR-ALS on the concatenation with G_N = [old; new] and old G_2..G_{N-1}
    c = [G.copy() for G in init[:-1]] + [st.cores[-1].copy()]
    als_mode_update(Xcat, c, 1)
    assert _rel(st.cores[0], c[0]) < 1e-10


def test_exact_stream_fixed_point_true_init():
    """Self-check 3 (primary): noise-free exact-rank stream (C1 shape), init = true cores:
    relative fit on the whole stream < 1e-8 after every batch."""
    cfg = make_stream("C1").cfg.with_(noise_abs=0.0, init_perturb=0.0)
    s = make_stream(cfg)
    st = StreamingTR(paper_view(s.init_slab()), s.init_cores())
    hist = [paper_view(s.init_slab())]
    for b in range(cfg.n_batches):
        Xb = paper_view(s.batch(b))
        st.update(Xb)
        hist.append(Xb)
        err = relative_error(np.concatenate(hist, axis=-1), st.cores)
        assert err < 1e-8, (b, err)


def test_exact_stream_fixed_point_als_init():
    """Self-check 3 (secondary): init by TR-ALS (Alg. 1) at tol 1e-12, init error <= 1e-10
    asserted, then tracking error < 1e-8 after every batch.  Retries another random start if
    ALS swamps."""
    cfg = make_stream("C1").cfg.with_(noise_abs=0.0)
    s = make_stream(cfg)
    Xi = paper_view(s.init_slab())
    for seed in range(8):
        rng = np.random.default_rng(100 + seed)
        R = cfg.ranks
        dims = cfg.dims + (cfg.t_init,)
        start = [rng.standard_normal((R[n], dims[n], R[(n + 1) % 3])) / np.sqrt(R[n] * R[(n + 1) % 3])
                 for n in range(3)]
        cores, err, _ = tr_als(Xi, R, start, tol=1e-14, max_sweeps=3000)
        if err <= 1e-10:
            break
    assert err <= 1e-10
    st = StreamingTR(Xi, cores)
    hist = [Xi]
    for b in range(cfg.n_batches):
        Xb = paper_view(s.batch(b))
        st.update(Xb)
        hist.append(Xb)
        assert relative_error(np.concatenate(hist, axis=-1), st.cores) < 1e-8


def test_Q_spd_and_monotone():
    """Q_n symmetric PSD and Q_n^after - Q_n^before PSD."""
    s = make_stream("T4")
    st = StreamingTR(paper_view(s.init_slab()), s.init_cores())
    for b in range(3):
        before = [q.copy() for q in st.Q]
        st.update(paper_view(s.batch(b)))
        for q0, q1 in zip(before, st.Q):
            assert np.allclose(q1, q1.T)
            assert np.linalg.eigvalsh(q1).min() > -1e-10 * np.trace(q1)
            assert np.linalg.eigvalsh(q1 - q0).min() > -1e-10 * np.trace(q1)


def test_memory_formula():
    """State scalars = (2(N-1)I + t_old) R^2 + (N-1) R^4, uniform I and R."""
    I, R, N, t = 5, 3, 4, 7
    cores = _cores((I,) * (N - 1) + (t,), (R,) * N, 3)
    X = np.random.default_rng(4).standard_normal((I,) * (N - 1) + (t,))
    st = StreamingTR(X, cores)
    assert st.state_scalars() == (2 * (N - 1) * I + t) * R ** 2 + (N - 1) * R ** 4


def test_blocked_contraction_equals_unblocked(monkeypatch):
    cores = _cores((4, 3, 5, 6), (2, 3, 4, 2), 5)
    X = np.random.default_rng(6).standard_normal((4, 3, 5, 6))
    full = [mode_n_times_subchain(X, cores, n) for n in range(1, 5)]
    monkeypatch.setattr(ost, "_BLOCK_ENTRIES", 1)
    for n in range(1, 5):
        np.testing.assert_allclose(mode_n_times_subchain(X, cores, n), full[n - 1], rtol=1e-13, atol=1e-13)


def test_fit_definition():
    """Fit: equals ||X - TR(G)||/||X|| by brute force; 0 on exact data; 1 with zero cores."""
    cores = _cores((3, 2, 4), (2, 3, 2), 7)
    X = tr_full_bruteforce(cores)
    assert relative_error(X, cores) < 1e-14
    noisy = X + 0.1 * np.random.default_rng(8).standard_normal(X.shape)
    ref = frobenius(noisy - X) / frobenius(noisy)
    assert abs(relative_error(noisy, cores) - ref) < 1e-13
    zero = [np.zeros_like(G) for G in cores]
    assert abs(relative_error(noisy, zero) - 1.0) < 1e-15
    with pytest.raises(ValueError):
        relative_error(np.zeros_like(X), cores)
