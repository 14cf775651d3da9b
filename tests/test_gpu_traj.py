"""Every-batch GPU parity at BASELINE.json's full sizes, including the TR-ALS initialization the
configs state, against the fp64 oracle.

C5 (the bench workload, 15 batches of 20.5M entries) is compared with oracle trajectories cached
by tests/golden/make_traj.py (a committed script that calls only oracle/ and workloads/; one
oracle step at C5 costs seconds): after EVERY batch, every non-temporal core, the new temporal
rows, the whole-stream fit, the per-row maximum relative error and the gauge-invariant
reconstruction difference of the latest batch (tests/_parity.py).  C2, C3 and C4 run the oracle
live from the cached TR-ALS init cores.  Tolerances (BASELINE.json north_star): 1e-9 with the FP64
contraction, 1e-4 with 3xTF32.  Per-row errors: 10x the core tolerance (a row's relative error
is that row's Frobenius error over its own norm, floored at 1e-3 of the rms row norm)."""
import os

import numpy as np
import pytest

from tests._parity import recon_rel, rel, row_rel
from workloads import make_stream
from workloads.gen import paper_view

TOL = {"f64": 1e-9, "3xtf32": 1e-4}
ROW = 10.0
TRAJ = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "traj")


def _als_init(name):
    d = np.load(os.path.join(TRAJ, f"{name}_als_init.npz"))
    n = sum(1 for k in d.files if k.startswith("core"))
    return [d[f"core{i}"] for i in range(1, n + 1)], float(d["err"]), int(d["sweeps"])


def _temporal_rows_paper(rows, RN, R1):
    """str_get_temporal_rows output (t x R_N R_1, column r_N + R_N r_1) -> paper layout R_N x t x R_1."""
    t = rows.shape[0]
    return rows.reshape(t, R1, RN).transpose(2, 0, 1)


def _c5_cached(contract, init):
    import torch
    import paper_2307_00719_b200 as lib
    path = os.path.join(TRAJ, f"C5_{init}_traj.npz")
    traj = np.load(path)
    s = make_stream("C5")
    cfg = s.cfg
    N, tol = cfg.N, TOL[contract]
    cores0 = _als_init("C5")[0] if init == "als" else s.init_cores()
    Xi = s.init_slab()
    hist = [torch.from_numpy(Xi).cuda()]
    h = lib.str_init(N, cfg.dims, cfg.ranks, hist[0], cfg.t_init, cores0, dtype=cfg.dtype, contract=contract,
                     split_k=cfg.split_k, t_capacity=cfg.T_total)
    RN, R1 = cfg.ranks[-1], cfg.ranks[0]
    report = []
    for b in range(cfg.n_batches):
        hist.append(torch.from_numpy(s.batch(b)).cuda())
        lib.str_update_batch(h, hist[-1], cfg.t_new)
        g = [lib.str_get_cores(h, n) for n in range(1, N)]
        o = [traj[f"b{b}_core{n}"] for n in range(1, N)]
        T = lib.str_processed(h)
        gnew = _temporal_rows_paper(lib.str_get_temporal_rows(h, T - cfg.t_new, cfg.t_new), RN, R1)
        onew = traj[f"b{b}_gnew"]
        errs = [rel(a, c) for a, c in zip(g, o)] + [rel(gnew, onew)]
        rows = [row_rel(a, c) for a, c in zip(g, o)] + [row_rel(gnew, onew)]
        fit_g = lib.str_fit(h, torch.cat(hist, dim=0), 0, T)
        fit_o = float(traj["fit"][b])
        rec = recon_rel(g + [gnew], o + [onew], 0, cfg.t_new) if (b % 5 == 4 or b == cfg.n_batches - 1) else None
        report.append((b, max(errs), max(rows), abs(fit_g - fit_o) / fit_o, rec))
        assert max(errs) <= tol, (contract, init, b, errs)
        assert max(rows) <= ROW * tol, (contract, init, b, rows)
        assert abs(fit_g - fit_o) <= tol * fit_o, (contract, init, b, fit_g, fit_o)
        if rec is not None:
            assert rec <= tol, (contract, init, b, rec)
    lib.str_destroy(h)
    print(f"\nC5 {contract} init={init} max cond(Q)={traj['condQ'].max():.3e}")
    for r in report:
        print("  batch %2d core %.2e row %.2e fit %.2e recon %s" % (r[0], r[1], r[2], r[3],
                                                                     "-" if r[4] is None else "%.2e" % r[4]))


@pytest.mark.gpu
@pytest.mark.parametrize("contract", ["3xtf32", "f64"])
@pytest.mark.parametrize("init", ["als", "pert"])
def test_C5_every_batch(contract, init):
    """configs[4] (the bench workload): all 15 batches, both contraction precisions, from the TR-ALS
    init of the stated protocol and from the bench's perturbed-truth init."""
    _c5_cached(contract, init)


def _live(name, contract, init_kind="als", fit_every=1):
    """Every batch against the live oracle; returns the per-batch metrics."""
    import torch
    import paper_2307_00719_b200 as lib
    from oracle.fit import relative_error
    from oracle.stream import StreamingTR
    s = make_stream(name)
    cfg = s.cfg
    N, tol = cfg.N, TOL[contract]
    cores0 = _als_init(name)[0] if init_kind == "als" else s.init_cores()
    Xi = s.init_slab()
    orc = StreamingTR(paper_view(Xi), cores0)
    hist_np = [Xi]
    hist = [torch.from_numpy(Xi).cuda()]
    h = lib.str_init(N, cfg.dims, cfg.ranks, hist[0], cfg.t_init, cores0, dtype=cfg.dtype, contract=contract,
                     split_k=cfg.split_k, t_capacity=cfg.T_total)
    worst = [0.0, 0.0, 0.0, 0.0]
    condq = 0.0
    for b in range(cfg.n_batches):
        Xb = s.batch(b)
        hist_np.append(Xb)
        hist.append(torch.from_numpy(Xb).cuda())
        lib.str_update_batch(h, hist[-1], cfg.t_new)
        orc.update(paper_view(Xb))
        condq = max(condq, max(np.linalg.cond(q) for q in orc.Q))
        g = [lib.str_get_cores(h, n) for n in range(1, N + 1)]
        errs = [rel(a, c) for a, c in zip(g, orc.cores)]
        rows = [row_rel(a, c) for a, c in zip(g, orc.cores)]
        assert max(errs) <= tol, (name, contract, b, errs)
        assert max(rows) <= ROW * tol, (name, contract, b, rows)
        worst[0] = max(worst[0], max(errs))
        worst[1] = max(worst[1], max(rows))
        if (b + 1) % fit_every == 0 or b == cfg.n_batches - 1:
            T = lib.str_processed(h)
            fo = relative_error(paper_view(np.concatenate(hist_np, axis=0)), orc.cores)
            fg = lib.str_fit(h, torch.cat(hist, dim=0), 0, T)
            assert abs(fg - fo) <= tol * fo, (name, contract, b, fg, fo)
            worst[2] = max(worst[2], abs(fg - fo) / fo)
            t0 = T - cfg.t_new
            rec = recon_rel([c if i < N - 1 else c[:, t0:, :] for i, c in enumerate(g)],
                            [c if i < N - 1 else c[:, t0:, :] for i, c in enumerate(orc.cores)], 0, cfg.t_new)
            assert rec <= tol, (name, contract, b, rec)
            worst[3] = max(worst[3], rec)
    lib.str_destroy(h)
    print(f"\n{name} {contract} init={init_kind}: max cond(Q)={condq:.3e} worst core {worst[0]:.2e} "
          f"row {worst[1]:.2e} fit {worst[2]:.2e} recon {worst[3]:.2e}")
    return worst, condq


@pytest.mark.gpu
def test_C3_als_init_every_batch_f64():
    """configs[2] from its TR-ALS init (cond(Q_n) reaches ~2e7): FP64 contraction, all 95 batches, 1e-9."""
    _live("C3", "f64", fit_every=5)


@pytest.mark.gpu
def test_C2_als_init_every_batch():
    """configs[1] from its TR-ALS init: 3xTF32, all 36 batches."""
    _live("C2", "3xtf32", fit_every=6)


@pytest.mark.gpu
def test_C4_als_init_every_batch():
    """configs[3] run as STR from its TR-ALS init: 3xTF32, all 19 batches."""
    _live("C4", "3xtf32", fit_every=5)
