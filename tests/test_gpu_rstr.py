"""GPU parity for rSTR-U / rSTR-L (Alg. 7, Alg. 8).

Uniform draws depend only on (seed, tau, k, I) and must be bit-identical between the C++ sampler
in libstr and the oracle's Python SplitMix64 (reading R11).  Leverage draws depend on
p_k computed on each side; the oracle replays the index tables the library reports
(str_get_index_table) and, separately, the oracle's own draws are compared (flips counted).
All rSTR arithmetic is fp64 on both sides: cores must agree to <= 1e-9 after every batch."""
import numpy as np
import pytest

from oracle.rstream import RandomizedStreamingTR
from oracle.sampler import draw_uniform, draw_weighted, leverage_distribution
from oracle.tralg import core_unfold
from workloads import get_config, make_stream
from workloads.gen import paper_view

TOL = 1e-9


def _run(name, kind, n_batches=None, seed=7):
    import torch
    import paper_2307_00719_b200 as lib
    s = make_stream(name)
    cfg = s.cfg
    m = cfg.sketch_rows
    N = cfg.N
    Xi = s.init_slab()
    init = s.init_cores()
    h = lib.str_init(N, cfg.dims, cfg.ranks, torch.from_numpy(Xi).cuda(), cfg.t_init, init, dtype=cfg.dtype,
                     contract="f64", variant=kind, sketch_rows=m, seed=seed)
    tables = {}
    for k in range(1, N + 1):
        tables[(0, k)] = lib.str_get_index_table(h, k, m).astype(np.int64)
    orc = RandomizedStreamingTR(paper_view(Xi), init, m, kind, seed, draw_hook=lambda tau, k, I, p: tables[(tau, k)])
    nb = cfg.n_batches if n_batches is None else n_batches
    out = []
    for b in range(nb):
        Xb = s.batch(b)
        lib.str_update_batch(h, torch.from_numpy(Xb).cuda(), cfg.t_new)
        for k in range(1, N + 1):
            tables[(b + 1, k)] = lib.str_get_index_table(h, k, m).astype(np.int64)
        orc.update(paper_view(Xb))
        errs = []
        for n in range(1, N + 1):
            g = lib.str_get_cores(h, n)
            o = orc.cores[n - 1]
            errs.append(np.linalg.norm(g - o) / np.linalg.norm(o))
        out.append(errs)
    return out, tables, orc


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["R4", "R5"])
def test_rstr_uniform_parity_and_bit_identical_draws(name):
    out, tables, orc = _run(name, "uniform")
    cfg = get_config(name)
    # C++ SplitMix64 == Python SplitMix64 for every (tau, k)
    for (tau, k), idx in tables.items():
        I = cfg.dims[k - 1] if k < cfg.N else (cfg.t_init if tau == 0 else cfg.t_new)
        np.testing.assert_array_equal(idx, draw_uniform(7, tau, k, cfg.N, I, cfg.sketch_rows))
    for b, errs in enumerate(out):
        assert max(errs) <= TOL, (b, errs)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["R4", "R5"])
def test_rstr_leverage_parity_replayed(name):
    out, tables, orc = _run(name, "leverage")
    for b, errs in enumerate(out):
        assert max(errs) <= TOL, (b, errs)
    # the oracle's own leverage draws from the replayed state: count index flips (expect 0 in fp64)
    cfg = get_config(name)
    flips = 0
    for k in range(1, cfg.N):
        p = leverage_distribution(core_unfold(orc.cores[k - 1]))
        own = draw_weighted(7, cfg.n_batches, k, cfg.N, p, cfg.sketch_rows)
        flips += int(np.sum(own != tables[(cfg.n_batches, k)]))
    assert flips == 0


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["uniform", "leverage"])
def test_rstr_C4_full_size(kind):
    """configs[3] (C4, 100^3, R=8, m=2000): all 19 batches at full size, cores <= 1e-9 (fp64 rSTR)."""
    out, tables, orc = _run("C4", kind)
    for b, errs in enumerate(out):
        assert max(errs) <= TOL, (b, errs)
