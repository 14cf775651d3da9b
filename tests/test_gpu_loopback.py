"""The library's sharded path (world_size > 1, X_new split along mode 1)
run on ONE GPU through an in-process loopback group: p handles, one per rank, whose collective
sites (C1 temporal partial, C2 left-mode partials and Z_1, C2' the pass-2 partial Y_R, the init
reductions) meet on the host and are summed by one plain kernel — the same library code the NCCL
path runs, with the collective backend swapped (comm.cu).  The p ranks' steps are captured into
one CUDA graph (strdbg_loopback_step) as in production replay, and every rank's cores are compared
after every batch with the cached oracle trajectory of C5 (tests/golden/traj, the unsharded fp64
oracle) — 1e-4 in 3xTF32 mode, 1e-9 in FP64 mode."""
import ctypes as C
import os
import threading

import numpy as np
import pytest

from tests._parity import rel
from workloads import make_stream

TRAJ = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "traj")
TOL = {"f64": 1e-9, "3xtf32": 1e-4}


def _shard(slab, p, r):
    w = slab.shape[-1] // p
    return np.ascontiguousarray(slab[..., r * w:(r + 1) * w])


def _run(p, contract, n_batches, graph=1):
    import torch
    import paper_2307_00719_b200 as lib
    traj = np.load(os.path.join(TRAJ, "C5_als_traj.npz"))
    d = np.load(os.path.join(TRAJ, "C5_als_init.npz"))
    cores0 = [d[f"core{i}"] for i in range(1, 6)]
    s = make_stream("C5")
    cfg = s.cfg
    N = cfg.N
    group = lib.str_loopback_create(p)
    Xi = s.init_slab()
    xi_d = [torch.from_numpy(_shard(Xi, p, r)).cuda() for r in range(p)]
    torch.cuda.synchronize()
    hs = [None] * p
    errs = [None] * p

    def init(r):   # str_init is collective: the ranks meet at the init reductions
        try:
            hs[r] = lib.str_init(N, cfg.dims, cfg.ranks, xi_d[r], cfg.t_init, cores0, dtype=cfg.dtype,
                                 contract=contract, split_k=cfg.split_k, t_capacity=cfg.T_total + 8,
                                 world_size=p, rank=r, loopback_group=group)
        except Exception as e:   # pragma: no cover
            errs[r] = e
    th = [threading.Thread(target=init, args=(r,)) for r in range(p)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert all(e is None for e in errs), errs
    f = lib._lib.lib.strdbg_loopback_step
    f.restype = C.c_int
    f.argtypes = [C.POINTER(C.c_void_p), C.c_int32, C.POINTER(C.c_void_p), C.c_int64, C.c_int32]
    hp = (C.c_void_p * p)(*[h.ptr.value if hasattr(h.ptr, "value") else h.ptr for h in hs])
    # fixed device buffers: the captured graph holds their addresses; each batch is copied in
    bufs = [torch.empty(_shard(s.batch(0), p, r).shape, dtype=torch.float32, device="cuda") for r in range(p)]
    xp = (C.c_void_p * p)(*[b.data_ptr() for b in bufs])
    worst = 0.0
    for b in range(n_batches):
        Xb = s.batch(b)
        for r in range(p):
            bufs[r].copy_(torch.from_numpy(_shard(Xb, p, r)))
        torch.cuda.synchronize()
        st = f(hp, p, xp, cfg.t_new, graph)
        assert st == 0, (st, lib.str_error_string(hs[0]))
        for r in range(p):
            lib.str_sync(hs[r])
        o = [traj[f"b{b}_core{n}"] for n in range(1, N)]
        for r in range(p):
            g = [lib.str_get_cores(hs[r], n) for n in range(1, N)]
            e = [rel(a, c) for a, c in zip(g, o)]
            T = lib.str_processed(hs[r])
            rows = lib.str_get_temporal_rows(hs[r], T - cfg.t_new, cfg.t_new)
            onew = traj[f"b{b}_gnew"]   # R_N x t x R_1 -> rows (t, r_N + R_N r_1)
            orows = onew.transpose(1, 2, 0).reshape(cfg.t_new, -1)
            e.append(rel(rows, orows))
            worst = max(worst, max(e))
            assert max(e) <= TOL[contract], (p, contract, b, r, e)
    for h in hs:
        lib.str_destroy(h)
    lib.str_loopback_destroy(group)
    return worst


@pytest.mark.gpu
@pytest.mark.parametrize("p", [2, 4, 8])
def test_loopback_sharded_C5_graph(p):
    """C5 (40 rows of mode 1 -> 20 / 10 / 5 per rank), 3xTF32, graph-captured, every batch."""
    w = _run(p, "3xtf32", 6)
    print(f"\nloopback p={p} 3xtf32: worst rel err {w:.2e}")


@pytest.mark.gpu
@pytest.mark.parametrize("contract,graph", [("f64", 1), ("3xtf32", 0), ("f64", 0)])
def test_loopback_sharded_C5_modes(contract, graph):
    """FP64 contraction and/or eager per-rank enqueue from p host threads (no graph), p = 4."""
    w = _run(4, contract, 3, graph=graph)
    print(f"\nloopback p=4 {contract} graph={graph}: worst rel err {w:.2e}")
