#!/usr/bin/env python
"""In-stream per-kernel timeline of str_update_batch (diagnostic; GPU only).

    python tools/timeline.py [--config C5] [--contract 3xtf32|f64] [--steps 10]

Records an event after every library launch (strdbg_timeline) and prints, per kernel name,
the summed time between consecutive events (the launch's in-stream duration including its
launch gap), per step.
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--contract", default=None)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--variant", default="det")
    a = ap.parse_args()
    import torch
    import paper_2307_00719_b200 as lib
    from workloads import get_config, make_stream
    cfg = get_config(a.config)
    s = make_stream(cfg)
    contract = a.contract or cfg.contract
    nd = min(4, cfg.n_batches)
    xs = [torch.from_numpy(s.batch(b)).cuda() for b in range(nd)]
    kw = {}
    if a.variant != "det":
        kw = dict(variant=a.variant, sketch_rows=cfg.sketch_rows or 2000, seed=1)
    h = lib.str_init(cfg.N, cfg.dims, cfg.ranks, torch.from_numpy(s.init_slab()).cuda(), cfg.t_init, s.init_cores(),
                     dtype=cfg.dtype, contract=contract, split_k=cfg.split_k,
                     t_capacity=cfg.t_init + cfg.t_new * (a.steps + 8), **kw)
    for i in range(3):
        lib.str_update_batch(h, xs[i % nd], cfg.t_new)
    lib.str_sync(h)
    L = lib._lib.lib
    L.strdbg_timeline.restype = C.c_int
    L.strdbg_timeline.argtypes = [C.c_void_p, C.c_int32]
    L.strdbg_timeline_dump.restype = C.c_int64
    L.strdbg_timeline_dump.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
    L.strdbg_timeline(h.ptr, 1)
    for i in range(a.steps):
        lib.str_update_batch(h, xs[i % nd], cfg.t_new)
    lib.str_sync(h)
    buf = C.create_string_buffer(1 << 16)
    L.strdbg_timeline_dump(h.ptr, buf, 1 << 16)
    rows = []
    for line in buf.value.decode().strip().splitlines():
        nm, ms, n = line.split()
        rows.append((float(ms), nm, int(n)))
    rows.sort(reverse=True)
    tot = sum(r[0] for r in rows)
    print(f"{cfg.name} {contract} {a.variant}: {1e3 * tot / a.steps:.1f} us/step over {a.steps} steps")
    print(f"{'kernel':28s} {'us/step':>9s} {'launch/step':>11s} {'us/launch':>9s} {'share':>6s}")
    for ms, nm, n in rows:
        print(f"{nm:28s} {1e3 * ms / a.steps:9.1f} {n / a.steps:11.1f} {1e3 * ms / n:9.2f} {100 * ms / tot:5.1f}%")
    L.strdbg_timeline(h.ptr, 0)
    lib.str_destroy(h)


if __name__ == "__main__":
    main()
