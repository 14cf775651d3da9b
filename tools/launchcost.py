#!/usr/bin/env python
"""Average time per back-to-back contraction launch (memset + kernel), C5 (diagnostic)."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2307_00719_b200 as lib
    from workloads import get_config, make_stream
    cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "C5")
    s = make_stream(cfg)
    X = torch.from_numpy(s.batch(0)).cuda()
    h = lib.str_init(cfg.N, cfg.dims, cfg.ranks, torch.from_numpy(s.init_slab()).cuda(), cfg.t_init, s.init_cores(),
                     dtype=cfg.dtype, contract="3xtf32", split_k=cfg.split_k)
    L = lib._lib.lib
    if os.environ.get("STR_TF_DBGFLAGS"):   # the diagnostic flags act only while the pipeline trace is on
        L.strdbg_tftrace.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_longlong)]
        L.strdbg_tftrace(h.ptr, 1, None)
    L.strdbg_contract_repeat.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.POINTER(C.c_double)]
    for pas in (1, 2):
        for reps in (1, 5, 20):
            ms = C.c_double(0)
            L.strdbg_contract_repeat(h.ptr, C.c_void_p(X.data_ptr()), pas, cfg.t_new, reps, C.byref(ms))
            print(f"pass {pas}: {reps:3d} back-to-back launches: {1e3 * ms.value:7.2f} us per launch")
    lib.str_destroy(h)


if __name__ == "__main__":
    main()
