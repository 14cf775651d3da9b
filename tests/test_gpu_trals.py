"""GPU batch TR-ALS (str_tr_als, Alg. 1) against the oracle.

The GPU sweeps update modes in the cyclic order N, 1..N-1 through Prop. 1 normal equations; the
oracle (oracle/als.py) solves each mode's LS problem with LAPACK lstsq on the materialized
subchain — an independent route to the same LS solutions.  After the sweeps the handle must
hold Alg. 4's init state for the fitted cores, so one more streamed batch is compared with the
oracle stream started from those cores.  Tolerances as for the stream: 1e-9 with the FP64
contraction, 1e-4 with 3xTF32 (BASELINE.json north_star)."""
import numpy as np
import pytest

from tests._parity import rel

CASES = [("P1", "f64", 1e-9), ("P3", "f64", 1e-9), ("P2", "3xtf32", 1e-4), ("P5", "3xtf32", 1e-4)]


@pytest.mark.gpu
@pytest.mark.parametrize("name,contract,tol", CASES)
def test_tr_als_sweeps_match_oracle(name, contract, tol):
    import torch
    import paper_2307_00719_b200 as lib
    from oracle.als import tr_als_sweep
    from oracle.fit import relative_error
    from oracle.stream import StreamingTR
    from workloads import make_stream
    from workloads.gen import paper_view

    s = make_stream(name)
    cfg = s.cfg
    N = cfg.N
    Xi = s.init_slab()
    Xi_d = torch.from_numpy(Xi).to("cuda")
    init = s.init_cores()
    h = lib.str_init(cfg.N, cfg.dims, cfg.ranks, Xi_d, cfg.t_init, init, dtype=cfg.dtype, contract=contract,
                     split_k=cfg.split_k)
    sweeps = 2
    fit_gpu = lib.str_tr_als(h, Xi_d, cfg.t_init, sweeps)
    X = paper_view(Xi)
    cores = [np.array(G) for G in init]
    order = [N] + list(range(1, N))
    for _ in range(sweeps):
        cores = tr_als_sweep(X, cores, order)
    errs = [rel(lib.str_get_cores(h, n), cores[n - 1]) for n in range(1, N + 1)]
    assert max(errs) <= tol, (name, errs)
    fit_orc = relative_error(X, cores)
    assert abs(fit_gpu - fit_orc) <= tol * max(fit_orc, 1e-3), (fit_gpu, fit_orc)
    assert lib.str_processed(h) == cfg.t_init
    # the rebuilt streaming state: one more batch against the oracle stream started from these cores
    orc = StreamingTR(X, cores)
    Xb = s.batch(0)
    lib.str_update_batch(h, torch.from_numpy(Xb).to("cuda"), cfg.t_new)
    orc.update(paper_view(Xb))
    errs = [rel(lib.str_get_cores(h, n), orc.cores[n - 1]) for n in range(1, N + 1)]
    assert max(errs) <= tol, (name, "after stream step", errs)
    lib.str_destroy(h)


@pytest.mark.gpu
def test_tr_als_lowers_the_fit_c2():
    """At full C2 size (60^3 x 20 init slab, 3xTF32): sweeps from the perturbed init reduce the
    relative error monotonically (ALS never increases the LS objective, Alg. 1)."""
    import torch
    import paper_2307_00719_b200 as lib
    from workloads import make_stream
    s = make_stream("C2")
    cfg = s.cfg
    Xi_d = torch.from_numpy(s.init_slab()).to("cuda")
    h = lib.str_init(cfg.N, cfg.dims, cfg.ranks, Xi_d, cfg.t_init, s.init_cores(), dtype=cfg.dtype,
                     contract=cfg.contract)
    f0 = lib.str_fit(h, Xi_d, 0, cfg.t_init)
    fits = [lib.str_tr_als(h, Xi_d, cfg.t_init, 1) for _ in range(3)]
    assert fits[0] <= f0 * (1 + 1e-6)
    assert all(b <= a * (1 + 1e-6) for a, b in zip(fits, fits[1:])), (f0, fits)
    lib.str_destroy(h)
