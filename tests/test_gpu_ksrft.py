"""GPU parity for rSTR-K (KSRFT, Alg. 9; readings R17-R22) against oracle/ksrft.py.

Index draws and sign flips are integer work on SplitMix64 streams (reading R11/R18): the library's
index tables must be bit-identical to the oracle's own draws.  Cores after every batch: <= 1e-9
relative with the fp64 mixing (contract "f64"), <= 1e-4 with the fp32 mixing that goes with the
3xTF32 contract (BASELINE.json north_star tolerance for the fp32 paths)."""
import numpy as np
import pytest

from oracle.ksrft import KSRFTStreamingTR
from workloads import make_stream
from workloads.gen import paper_view


def _run(name, contract, n_batches, seed=7, m=None):
    import torch
    import paper_2307_00719_b200 as lib
    s = make_stream(name)
    cfg = s.cfg
    m = m or cfg.sketch_rows
    N = cfg.N
    Xi = s.init_slab()
    init = s.init_cores()
    h = lib.str_init(N, cfg.dims, cfg.ranks, torch.from_numpy(Xi).cuda(), cfg.t_init, init, dtype=cfg.dtype,
                     contract=contract, variant="ksrft", sketch_rows=m, seed=seed)
    orc = KSRFTStreamingTR(paper_view(Xi), init, m, seed)
    for k in range(1, N + 1):
        np.testing.assert_array_equal(lib.str_get_index_table(h, k, m), orc.draws[(0, k)])
    errs = []
    for b in range(n_batches):
        Xb = s.batch(b)
        lib.str_update_batch(h, torch.from_numpy(Xb).cuda(), cfg.t_new)
        orc.update(paper_view(Xb))
        for k in range(1, N + 1):
            np.testing.assert_array_equal(lib.str_get_index_table(h, k, m), orc.draws[(b + 1, k)])
        e = []
        for n in range(1, N + 1):
            g = lib.str_get_cores(h, n)
            o = orc.cores[n - 1]
            e.append(float(np.linalg.norm(g - o) / np.linalg.norm(o)))
        errs.append(e)
    lib.str_destroy(h)
    return errs


@pytest.mark.gpu
@pytest.mark.parametrize("name,contract,tol", [("R4", "f64", 1e-9), ("R5", "f64", 1e-9), ("R4", "3xtf32", 1e-4),
                                               ("R5", "3xtf32", 1e-4)])
def test_rstrk_parity(name, contract, tol):
    errs = _run(name, contract, 3)
    assert max(max(e) for e in errs) <= tol, errs


@pytest.mark.gpu
@pytest.mark.parametrize("contract,tol", [("f64", 1e-9), ("3xtf32", 1e-4)])
def test_rstrk_ragged_dims_and_prime_modes(contract, tol):
    """Mode lengths with no factorization (prime 17, 19: the generic mixing kernel's direct sums),
    24 = 4 x 6 and t_new = 5 (compile-time p x q kernels on the fp32 path); ragged tiles."""
    errs = _run("P2", contract, 2, m=300)
    assert max(max(e) for e in errs) <= tol, errs


@pytest.mark.gpu
def test_rstrk_full_size_c4():
    """BASELINE config C4 (100^3 x 10 per batch, R = 8, m = 2000) with the bench's launch
    configuration (fp32 mixing, graph replay): all 19 batches against the oracle."""
    errs = _run("C4", "3xtf32", 19)
    assert max(max(e) for e in errs) <= 1e-4, errs


@pytest.mark.gpu
def test_rstrk_graph_replay_is_deterministic():
    import torch
    import paper_2307_00719_b200 as lib
    s = make_stream("R4")
    cfg = s.cfg
    out = []
    for _ in range(2):
        h = lib.str_init(cfg.N, cfg.dims, cfg.ranks, torch.from_numpy(s.init_slab()).cuda(), cfg.t_init,
                         s.init_cores(), dtype=cfg.dtype, contract="3xtf32", variant="ksrft",
                         sketch_rows=cfg.sketch_rows, seed=11)
        for b in range(3):
            lib.str_update_batch(h, torch.from_numpy(s.batch(b)).cuda(), cfg.t_new)
        out.append([lib.str_get_cores(h, n) for n in range(1, cfg.N + 1)])
        lib.str_destroy(h)
    for a, b in zip(*out):
        np.testing.assert_array_equal(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("contract,tol", [("f64", 1e-9), ("3xtf32", 1e-4)])
def test_rstrk_varying_t_new_and_single_slice(contract, tol):
    """t_new = 3, 1, 4, 1, 2 (F_N of size 1 is the identity up to the sign flip; every new t_new
    re-captures the step graph; the sign stream length changes with t_new)."""
    import torch
    import paper_2307_00719_b200 as lib
    s = make_stream("R5")
    cfg = s.cfg
    m, N, seed = cfg.sketch_rows, cfg.N, 5
    h = lib.str_init(N, cfg.dims, cfg.ranks, torch.from_numpy(s.init_slab()).cuda(), cfg.t_init, s.init_cores(),
                     dtype=cfg.dtype, contract=contract, variant="ksrft", sketch_rows=m, seed=seed, t_capacity=64)
    orc = KSRFTStreamingTR(paper_view(s.init_slab()), s.init_cores(), m, seed)
    t0 = cfg.t_init
    for tn in (3, 1, 4, 1, 2):
        slab = np.ascontiguousarray(s.slab(t0, tn))
        t0 += tn
        lib.str_update_batch(h, torch.from_numpy(slab).cuda(), tn)
        orc.update(paper_view(slab))
        np.testing.assert_array_equal(lib.str_get_index_table(h, N, m), orc.draws[(orc.tau, N)])
        for n in range(1, N + 1):
            g, o = lib.str_get_cores(h, n), orc.cores[n - 1]
            assert np.linalg.norm(g - o) / np.linalg.norm(o) <= tol, (tn, n)
    lib.str_destroy(h)


@pytest.mark.gpu
def test_rstrk_host_draws_and_replayed_tables(monkeypatch):
    """The host sampler (STR_RSTR_HOST_DRAWS=1: host index draws, eager steps) gives the same
    tables and cores as the oracle; the sign flips stay on the device."""
    import torch
    import paper_2307_00719_b200 as lib
    monkeypatch.setenv("STR_RSTR_HOST_DRAWS", "1")
    s = make_stream("R4")
    cfg = s.cfg
    m, N = cfg.sketch_rows, cfg.N
    h = lib.str_init(N, cfg.dims, cfg.ranks, torch.from_numpy(s.init_slab()).cuda(), cfg.t_init, s.init_cores(),
                     dtype=cfg.dtype, contract="f64", variant="ksrft", sketch_rows=m, seed=9)
    orc = KSRFTStreamingTR(paper_view(s.init_slab()), s.init_cores(), m, 9)
    for b in range(2):
        lib.str_update_batch(h, torch.from_numpy(s.batch(b)).cuda(), cfg.t_new)
        orc.update(paper_view(s.batch(b)))
    errs = [np.linalg.norm(lib.str_get_cores(h, n) - orc.cores[n - 1]) / np.linalg.norm(orc.cores[n - 1])
            for n in range(1, N + 1)]
    assert max(errs) <= 1e-9, errs
    lib.str_destroy(h)


@pytest.mark.gpu
def test_rstrk_forced_index_tables():
    """Index tables forced through str_set_index_table (for every draw of each mode) against the
    oracle with the same tables injected by its draw hook; sign flips still from the seed."""
    import torch
    import paper_2307_00719_b200 as lib
    s = make_stream("R4")
    cfg = s.cfg
    m, N = cfg.sketch_rows, cfg.N
    rng = np.random.default_rng(12)
    lim = list(cfg.dims) + [min(cfg.t_init, cfg.t_new)]
    tables = {k: rng.integers(0, lim[k - 1], m).astype(np.int32) for k in range(1, N + 1)}
    # the init draws come from the seed (str_init draws before a table can be set); updates are forced
    h = lib.str_init(N, cfg.dims, cfg.ranks, torch.from_numpy(s.init_slab()).cuda(), cfg.t_init, s.init_cores(),
                     dtype=cfg.dtype, contract="f64", variant="ksrft", sketch_rows=m, seed=4)
    init_tabs = {k: lib.str_get_index_table(h, k, m).astype(np.int64) for k in range(1, N + 1)}
    for k in range(1, N + 1):
        lib.str_set_index_table(h, k, tables[k])
    orc = KSRFTStreamingTR(paper_view(s.init_slab()), s.init_cores(), m, 4,
                           draw_hook=lambda tau, k, I, p: init_tabs[k] if tau == 0 else tables[k])
    for b in range(2):
        lib.str_update_batch(h, torch.from_numpy(s.batch(b)).cuda(), cfg.t_new)
        orc.update(paper_view(s.batch(b)))
        for k in range(1, N + 1):
            np.testing.assert_array_equal(lib.str_get_index_table(h, k, m), tables[k])
    errs = [np.linalg.norm(lib.str_get_cores(h, n) - orc.cores[n - 1]) / np.linalg.norm(orc.cores[n - 1])
            for n in range(1, N + 1)]
    assert max(errs) <= 1e-9, errs
    lib.str_destroy(h)
