"""rSTR probe (diagnostic): init a C4 rSTR handle (variant: ksrft / uniform / leverage) and run a
few steps (for ncu).   python tools/ks_probe.py [config] [steps] [variant]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2307_00719_b200 as lib  # noqa: E402
from workloads import get_config, make_stream  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "C4")
s = make_stream(cfg)
variant = sys.argv[3] if len(sys.argv) > 3 else "ksrft"
h = lib.str_init(cfg.N, cfg.dims, cfg.ranks, torch.from_numpy(s.init_slab()).cuda(), cfg.t_init, s.init_cores(),
                 dtype=cfg.dtype, contract="3xtf32", variant=variant, sketch_rows=cfg.sketch_rows or 2000, seed=1)
x = torch.from_numpy(s.batch(0)).cuda()
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    lib.str_update_batch(h, x, cfg.t_new)
lib.str_sync(h)
print("ok")
