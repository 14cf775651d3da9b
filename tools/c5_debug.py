"""Repeated C5 runs with a sync + finiteness check after every step (diagnostic; GPU only)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_00719_b200 as lib
from workloads import get_config, make_stream
cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "C5")
contract = sys.argv[2] if len(sys.argv) > 2 else cfg.contract
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 12
s = make_stream(cfg)
xs = [torch.from_numpy(s.batch(b)).cuda() for b in range(8)]
for trial in range(3):
    h = lib.str_init(cfg.N, cfg.dims, cfg.ranks, torch.from_numpy(s.init_slab()).cuda(), cfg.t_init, s.init_cores(),
                     dtype=cfg.dtype, contract=contract, split_k=cfg.split_k, t_capacity=2000)
    ok = True
    for st in range(steps):
        lib.str_update_batch(h, xs[st % 8], cfg.t_new)
        try:
            lib.str_sync(h)
        except Exception as e:
            print(f"trial {trial} step {st}: {e}")
            ok = False
            break
        bad = [n for n in range(1, cfg.N + 1) if not np.isfinite(lib.str_get_cores(h, n)).all()]
        if bad:
            print(f"trial {trial} step {st}: non-finite cores {bad}")
            ok = False
            break
    print(f"trial {trial}: {'ok' if ok else 'FAILED'}", flush=True)
    lib.str_destroy(h)
