#!/usr/bin/env python
"""Pipeline trace of the tensor-core contraction (CTA 0): per unit, cycles relative to the first
producer event: [0] producer X issue, [1] conv X landed, [2] conv A slot free, [3] conv done,
[4] MMA B landed, [5] MMA A ready, [6] MMA issued.  Diagnostic; GPU only."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2307_00719_b200 as lib
    from workloads import get_config, make_stream
    name = sys.argv[1] if len(sys.argv) > 1 else "C5"
    pas = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    cfg = get_config(name)
    s = make_stream(cfg)
    # distinct batches per run so that X streams from HBM as in the bench (82 MB each > L2 / 2)
    Xs = [torch.from_numpy(s.batch(b % cfg.n_batches)).cuda() for b in range(4)]
    h = lib.str_init(cfg.N, cfg.dims, cfg.ranks, torch.from_numpy(s.init_slab()).cuda(), cfg.t_init, s.init_cores(),
                     dtype=cfg.dtype, contract="3xtf32", split_k=cfg.split_k)
    L = lib._lib.lib
    L.strdbg_tftrace.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_longlong)]
    L.strdbg_contract.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double)]
    out = np.zeros(20_000_000)
    for it in range(4):
        X = Xs[it]
        L.strdbg_tftrace(h.ptr, 1, None)
        L.strdbg_contract(h.ptr, C.c_void_p(X.data_ptr()), pas, min(cfg.t_new, cfg.t_init),
                          out.ctypes.data_as(C.POINTER(C.c_double)))
        W = 1024 + 4 * 160
        tr2 = np.zeros(2 * W, dtype=np.int64)
        L.strdbg_tftrace(h.ptr, 0, tr2.ctypes.data_as(C.POINTER(C.c_longlong)))
        tr = tr2[(pas - 1) * W:pas * W]
    g = tr[1024:].reshape(160, 4)
    g = g[g[:, 0] > 0]
    t00 = g[:, 0].min()
    gg = (g - t00) / 1000.0
    print(f"CTAs: {len(g)}; us rel. to first CTA entry: entry max {gg[:,0].max():.2f}, setup done max "
          f"{gg[:,1].max():.2f}, last MMA issued min/med/max {gg[:,2].min():.2f}/{np.median(gg[:,2]):.2f}/"
          f"{gg[:,2].max():.2f}, exit min/med/max {gg[:,3].min():.2f}/{np.median(gg[:,3]):.2f}/{gg[:,3].max():.2f}")
    tr = tr[:1024].reshape(64, 16)
    if os.environ.get("STR_TF_DBGFLAGS", "0").isdigit() and int(os.environ.get("STR_TF_DBGFLAGS", "0")) & 256:
        print(f"bare MMA loop inside the kernel: {tr[63, 0]} cycles for the CTA's units")
        return
    n = int((tr[:, 6] > 0).sum())
    t0 = tr[0, 0]
    print(f"{name} pass {pas}: {n} units traced (cycles rel. to first X issue)")
    print("unit  Xissue  Bissue  Xlanded  Aslot  convdone  Bready  Aready  MMAissued  committed  dMMA")
    prev = None
    for u in range(n):
        r = tr[u] - t0
        d = "" if prev is None else str(r[6] - prev)
        print(f"{u:4d} {r[0]:7d} {r[8]:7d} {r[1]:8d} {r[2]:6d} {r[3]:9d} {r[4]:7d} {r[5]:7d} {r[6]:9d} {r[7]:9d} {d:>6s}")
        prev = r[6]


if __name__ == "__main__":
    main()
