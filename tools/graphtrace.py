#!/usr/bin/env python
"""Per-CTA globaltimer spans of the two contraction passes inside the replayed step graph (C5 by
default): kernel start-to-end, CTA entry spread, last-MMA and exit distributions.  Diagnostic."""
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
    cfg = get_config(name)
    s = make_stream(cfg)
    xs = [torch.from_numpy(s.batch(b)).cuda() for b in range(6)]
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        h = lib.str_init(cfg.N, cfg.dims, cfg.ranks, torch.from_numpy(s.init_slab()).cuda(), cfg.t_init,
                         s.init_cores(), dtype=cfg.dtype, contract=cfg.contract, split_k=cfg.split_k,
                         t_capacity=cfg.t_init + cfg.t_new * 40, stream=stream.cuda_stream)
    L = lib._lib.lib
    L.strdbg_tftrace.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_longlong)]
    L.strdbg_tftrace(h.ptr, 1, None)
    prof = "--prof" in sys.argv
    if prof:
        lib.str_set_profiling(h, True)
    for i in range(12):
        lib.str_update_batch(h, xs[i % 6], cfg.t_new)
    lib.str_sync(h)
    if prof:
        p1, n1, p2, n2 = lib.str_profile(h)
        print(f"events (profiling graph): pass 1 {1e3 * p1 / max(n1, 1):.2f} us, pass 2 {1e3 * p2 / max(n2, 1):.2f} us")
    W = 1024 + 4 * 160
    tr = np.zeros(2 * W, dtype=np.int64)
    L.strdbg_tftrace(h.ptr, 0, tr.ctypes.data_as(C.POINTER(C.c_longlong)))
    base = None
    for pas in (1, 2):
        g = tr[(pas - 1) * W + 1024:pas * W].reshape(160, 4)
        g = g[g[:, 0] > 0].astype(np.float64)
        if base is None:
            base = g[:, 0].min()
        e0 = g[:, 0].min()
        rel = (g - e0) / 1e3
        span = (g[:, 3].max() - e0) / 1e3
        ok = g[:, 2] > 0
        print(f"pass {pas}: starts {1e-3 * (e0 - base):8.2f} us after pass 1; span {span:6.2f} us; CTAs {len(g)}")
        for k, nm in ((0, "entry"), (1, "setup"), (2, "lastMMA"), (3, "exit")):
            col = rel[ok, k] if k == 2 else rel[:, k]
            print(f"   {nm:8s} min/p10/med/p90/max {col.min():7.2f} {np.percentile(col, 10):7.2f} {np.median(col):7.2f} "
                  f"{np.percentile(col, 90):7.2f} {col.max():7.2f}")
    lib.str_destroy(h)


if __name__ == "__main__":
    main()
