"""A few rSTR-U / STR steps at C4 for ncu captures of the small kernels (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2307_00719_b200 as lib  # noqa: E402
from workloads import get_config, make_stream  # noqa: E402

variant = sys.argv[1] if len(sys.argv) > 1 else "uniform"
cfg = get_config("C4")
s = make_stream(cfg)
xs = [torch.from_numpy(s.batch(b)).cuda() for b in range(3)]
kw = dict(variant=variant, sketch_rows=2000, seed=1) if variant != "det" else {}
h = lib.str_init(cfg.N, cfg.dims, cfg.ranks, torch.from_numpy(s.init_slab()).cuda(), cfg.t_init, s.init_cores(),
                 dtype=cfg.dtype, contract=cfg.contract, **kw)
for i in range(3):
    lib.str_update_batch(h, xs[i], cfg.t_new)
lib.str_sync(h)
print("ok")
