"""GPU edge cases of the STR step (Alg. 4) against the oracle: single-slice and varying batches,
degenerate ranks (R_1 = 1: the ring closes through a rank-1 bond, i.e. a tensor train, the TT
case of Remark P:400-403), a mode of length 1, and the error contract on a live handle."""
import numpy as np
import pytest

from oracle.stream import StreamingTR
from tests._parity import rel
from workloads import get_config, make_stream
from workloads.gen import paper_view

TOL = {"f64": 1e-9, "3xtf32": 1e-4}


def _run_sequence(cfg, contract, t_seq):
    import torch
    import paper_2307_00719_b200 as lib
    s = make_stream(cfg)
    Xi = s.init_slab()
    init = s.init_cores()
    h = lib.str_init(cfg.N, cfg.dims, cfg.ranks, torch.from_numpy(Xi).cuda(), cfg.t_init, init, dtype=cfg.dtype,
                     contract=contract, split_k=cfg.split_k, t_capacity=cfg.t_init + sum(t_seq) + 4)
    orc = StreamingTR(paper_view(Xi), init)
    t0 = cfg.t_init
    worst = 0.0
    for tn in t_seq:
        slab = np.ascontiguousarray(s.slab(t0, tn))
        t0 += tn
        lib.str_update_batch(h, torch.from_numpy(slab).cuda(), tn)
        orc.update(paper_view(slab))
        errs = [rel(lib.str_get_cores(h, n), orc.cores[n - 1]) for n in range(1, cfg.N + 1)]
        worst = max(worst, max(errs))
        assert max(errs) <= TOL[contract], (tn, errs)
    assert lib.str_processed(h) == t0
    lib.str_destroy(h)
    return worst


@pytest.mark.gpu
@pytest.mark.parametrize("contract", ["f64", "3xtf32"])
def test_varying_t_new_incl_single_slices(contract):
    """t_new = 5, 1, 3, 1, 7, 2: every new t_new re-captures the step graph (pass-1 M-tiles pair
    across t, so odd and single-slice batches exercise the unpaired tile)."""
    _run_sequence(get_config("P2"), contract, (5, 1, 3, 1, 7, 2))


@pytest.mark.gpu
@pytest.mark.parametrize("contract", ["f64", "3xtf32"])
def test_rank_one_bond_tensor_train(contract):
    """R_1 = 1 (TT as a TR with one rank-1 bond): R_N R_1 = 3 temporal columns, rank-1 chain factors."""
    cfg = get_config("P2").with_(name="P2-TT", ranks=(1, 4, 5, 3))
    _run_sequence(cfg, contract, (5, 5))


@pytest.mark.gpu
def test_mode_of_length_one():
    """I_2 = 1: a degenerate mode (its core is a single R_2 x R_3 slice).  R_2 = R_3 keeps that slice
    square: with R_2 < R_3 the subchains through it have rank <= R_2 R_{n+1} < R_3 R_{n+1}, Q_n is
    exactly singular and the LS solution is not unique (the oracle's pseudo-inverse picks the
    minimum-norm one, reading R3), so only the full-rank case has a unique answer to compare."""
    cfg = get_config("P2").with_(name="P2-I1", dims=(24, 1, 17), ranks=(3, 4, 4, 2))
    _run_sequence(cfg, "f64", (5, 2))


@pytest.mark.gpu
def test_error_contract_on_a_live_handle():
    import torch
    import paper_2307_00719_b200 as lib
    from paper_2307_00719_b200._lib import STR_E_ARG, StrError
    s = make_stream("T4")
    cfg = s.cfg
    h = lib.str_init(cfg.N, cfg.dims, cfg.ranks, torch.from_numpy(s.init_slab()).cuda(), cfg.t_init,
                     s.init_cores(), dtype=cfg.dtype, contract="f64")
    Xb = torch.from_numpy(s.batch(0)).cuda()
    import ctypes as C                          # t_new >= 1, at the C boundary itself
    assert lib._lib.lib.str_update_batch(h.ptr, C.c_void_p(Xb.data_ptr()), 0) == STR_E_ARG
    assert lib._lib.lib.str_update_batch(h.ptr, None, cfg.t_new) == STR_E_ARG
    with pytest.raises(StrError) as e:          # ||X|| = 0 is an error for the fit
        lib.str_fit(h, torch.zeros_like(Xb), 0, cfg.t_new)
    assert e.value.status == STR_E_ARG
    with pytest.raises(StrError):               # rows beyond what has been processed
        lib.str_get_temporal_rows(h, lib.str_processed(h), 1)
    with pytest.raises(StrError):               # index tables exist only for rSTR handles
        lib.str_get_index_table(h, 1, 4)
    # the handle is still usable after argument errors (they do not poison it)
    lib.str_update_batch(h, Xb, cfg.t_new)
    assert lib.str_processed(h) == cfg.t_init + cfg.t_new
    lib.str_destroy(h)
