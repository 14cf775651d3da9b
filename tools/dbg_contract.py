import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2307_00719_b200 as lib
from workloads import make_stream
from tests.test_gpu_contract import _chain
name = sys.argv[1] if len(sys.argv) > 1 else "P2"
for contract in ("f64", "3xtf32"):
    for pass_ in (1, 2):
        s = make_stream(name); cfg = s.cfg; Xi = s.init_slab()
        h = lib.str_init(cfg.N, cfg.dims, cfg.ranks, torch.from_numpy(Xi).cuda(), cfg.t_init, s.init_cores(), dtype=cfg.dtype, contract=contract, split_k=cfg.split_k)
        N = cfg.N; k = cfg.split_k or 1; tn = cfg.t_init
        L = int(np.prod(cfg.dims[:k])); Rr = int(np.prod(cfg.dims[k:])); W = cfg.ranks[k] * cfg.ranks[N-1]
        out = np.empty((L*tn if pass_ == 1 else Rr) * W)
        fn = lib._lib.lib.strdbg_contract; fn.restype = C.c_int
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double)]
        Xd = torch.from_numpy(Xi).cuda()
        st = fn(h.ptr, C.c_void_p(Xd.data_ptr()), pass_, tn, out.ctypes.data_as(C.POINTER(C.c_double)))
        print(contract, "pass", pass_, "status", st, lib.str_error_string(h), "L", L, "Rr", Rr, "W", W)
        o = out.reshape(-1, W)
        print("  nonzeros", np.count_nonzero(o), "of", o.size, "norm", np.linalg.norm(o))
        print("  row0", np.round(o[0, :8], 4))
        print("  row1", np.round(o[1, :8], 4))
        print("  row130", np.round(o[min(130, o.shape[0]-1), :8], 4))
