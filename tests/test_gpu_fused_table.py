"""Pass 2 with the table formed inside the tcgen05 contraction kernel (the fused subchain generation
of BASELINE.json's north_star; Def. 3, Alg. 4 l.13-14 P:375-376): every batch against the
fp64 oracle, and the path selection itself.

The kernel's generator warps multiply each K-tile's prefix rows F = G_N(t) G_1(i_1) ... G_{k-1}
by G_k(i_k) in fp32 and split the product into tf32 hi / lo in shared memory, so T_L never exists
in HBM.  G4 / G10 have K-tiles that cross a multiple of I_1 (two prefix-row runs and two G_k
slices per tile), G8 has I_1 = 32 (every tile aligned); all have a ragged last K-tile and M-tile.
The path is opt-in per handle (STR_TF_GEN=1 when str_init runs): it measured slower than the
pre-tiled table at C5, so production keeps the table kernel."""
import ctypes as C

import pytest

from tests._parity import gpu_stream

TOL = 1e-4   # 3xTF32 mode (BASELINE.json north_star)


def _gen_rank(h):
    import paper_2307_00719_b200 as lib
    f = lib._lib.lib.strdbg_tf32_gen_rank
    f.restype = C.c_int32
    f.argtypes = [C.c_void_p]
    return f(h.ptr)


@pytest.mark.gpu
@pytest.mark.parametrize("name,rank", [("G4", 4), ("G8", 8), ("G10", 10)])
def test_fused_pass2_every_batch(name, rank, monkeypatch):
    monkeypatch.setenv("STR_TF_GEN", "1")
    for b, errs, fo, fg, h, orc in gpu_stream(name, contract="3xtf32"):
        assert _gen_rank(h) == rank
        assert max(errs) <= TOL, (b, errs)
        assert abs(fg - fo) <= TOL * fo, (b, fo, fg)


@pytest.mark.gpu
@pytest.mark.parametrize("name,contract,split_k", [("P5", "3xtf32", 2), ("G10", "f64", 2), ("G10", "3xtf32", 1)])
def test_fused_path_not_taken(name, contract, split_k, monkeypatch):
    """Non-uniform ranks, the FP64 contraction, or k = 1 keep the pre-tiled table (and stay exact)."""
    monkeypatch.setenv("STR_TF_GEN", "1")
    for b, errs, fo, fg, h, orc in gpu_stream(name, contract=contract, split_k=split_k, n_batches=1):
        assert _gen_rank(h) == 0
        assert max(errs) <= (1e-9 if contract == "f64" else TOL), (b, errs)


@pytest.mark.gpu
def test_fused_path_off_by_default(monkeypatch):
    monkeypatch.delenv("STR_TF_GEN", raising=False)
    for b, errs, fo, fg, h, orc in gpu_stream("G10", contract="3xtf32", n_batches=1):
        assert _gen_rank(h) == 0
        assert max(errs) <= TOL, (b, errs)
