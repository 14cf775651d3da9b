"""GPU unit tests of the two contraction passes (the dominant kernels) against a numpy fp64
evaluation of the same grouped products (Def. 3 subchain slices):
  pass 1: Y_L[(l,t)] = sum_r X[l, r, t] (G_{k+1} ... G_{N-1})(r)
  pass 2: Y_R[r]     = sum_{l,t} X[l, r, t] (G_N(t) G_1 ... G_k)(l)
Tolerances: 1e-12 (FP64 path), 2e-6 relative Frobenius (3xTF32 path)."""
import ctypes as C

import numpy as np
import pytest

from workloads import make_stream

TOL = {"f64": 1e-12, "3xtf32": 2e-6}


def _chain(cores, modes):
    """Row-major products over the multi-index of `modes` (first mode fastest)."""
    T = None
    for n in modes:
        S = cores[n - 1].transpose(1, 0, 2)          # (I, Ra, Rb)
        if T is None:
            T = S
        else:
            T = np.einsum("xab,ybc->yxac", T, S).reshape(-1, T.shape[1], S.shape[2])
    return T


def _run(name, contract, pass_):
    import torch
    import paper_2307_00719_b200 as lib
    s = make_stream(name)
    cfg = s.cfg
    Xi = s.init_slab()
    h = lib.str_init(cfg.N, cfg.dims, cfg.ranks, torch.from_numpy(Xi).cuda(), cfg.t_init, s.init_cores(),
                     dtype=cfg.dtype, contract=contract, split_k=cfg.split_k)
    N = cfg.N
    cores = [lib.str_get_cores(h, n) for n in range(1, N + 1)]
    k = cfg.split_k or 1
    tn = cfg.t_init
    Xp = Xi.astype(np.float64).reshape(tn, -1)                  # (t, slice) paper order per slice
    L = int(np.prod(cfg.dims[:k]))
    Rr = int(np.prod(cfg.dims[k:]))
    X3 = Xp.reshape(tn, Rr, L)                                   # [t][r][l]
    W = cfg.ranks[k] * cfg.ranks[N - 1]
    out = np.empty((L * tn if pass_ == 1 else Rr) * W)
    fn = lib._lib.lib.strdbg_contract
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double)]
    Xd = torch.from_numpy(Xi).cuda()
    st = fn(h.ptr, C.c_void_p(Xd.data_ptr()), pass_, tn, out.ctypes.data_as(C.POINTER(C.c_double)))
    assert st == 0, lib.str_error_string(h)
    if pass_ == 1:
        TR = _chain(cores, list(range(k + 1, N))).reshape(Rr, W)              # (Rr, W)
        ref = np.einsum("trl,rw->tlw", X3, TR).reshape(L * tn, W)
    else:
        GN = cores[-1].transpose(1, 0, 2)[:tn]                                  # (t, R_N, R_1)
        CL = _chain(cores, list(range(1, k + 1)))                               # (L, R_1, R_{k+1})
        TL = np.einsum("tab,lbc->tlac", GN, CL).reshape(tn * L, W)              # row l + L t
        ref = np.einsum("trl,tlw->rw", X3, TL.reshape(tn, L, W))
    got = out.reshape(ref.shape)
    return np.linalg.norm(got - ref) / np.linalg.norm(ref)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["P2", "P5", "T4"])
@pytest.mark.parametrize("pass_", [1, 2])
def test_contract_f64(name, pass_):
    assert _run(name, "f64", pass_) < TOL["f64"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["P2", "P5", "G4", "G8", "G10"])
@pytest.mark.parametrize("pass_", [1, 2])
def test_contract_3xtf32(name, pass_):
    assert _run(name, "3xtf32", pass_) < TOL["3xtf32"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["G4", "G8", "G10"])
def test_contract_3xtf32_fused_pass2(name, monkeypatch):
    """Pass 2 with its table formed inside the contraction kernel (opt-in STR_TF_GEN=1 at str_init)."""
    monkeypatch.setenv("STR_TF_GEN", "1")
    assert _run(name, "3xtf32", 2) < TOL["3xtf32"]
