"""The C-ABI's argument validation (include/str.h), exercised without a GPU: every invalid
configuration must be rejected by str_init with the documented status before any CUDA work, and
every entry point must reject a NULL handle.  SPEC S:404 (t >= 1), S:451 (m >= R_nR_{n+1})."""
import ctypes as C

import pytest

from paper_2307_00719_b200 import _lib as L

FAKE = C.c_void_p(64)   # non-NULL, never dereferenced: validation fails first


def _cfg(order=4, dims=(6, 5, 4), ranks=(2, 3, 2, 2), dtype=L.STR_F32, contract=L.STR_CONTRACT_F64,
         variant=L.STR_DET, m=0, split_k=0, world=1, rank=0):
    d = (C.c_int64 * len(dims))(*dims)
    r = (C.c_int32 * len(ranks))(*ranks)
    cfg = L.str_config(order=order, dims=d, ranks=r, dtype=dtype, contract=contract, variant=variant,
                       sketch_rows=m, seed=1, t_capacity=0, split_k=split_k, world_size=world, rank=rank,
                       nccl_id=None, device=0, stream=None)
    return cfg, (d, r)


def _init(cfg, t_init=3):
    cores = (C.POINTER(C.c_double) * 8)(*[C.cast(FAKE, C.POINTER(C.c_double))] * 8)
    out = C.c_void_p()
    st = L.lib.str_init(C.byref(cfg), FAKE, t_init, cores, C.byref(out))
    assert not out.value   # nothing is created on a rejected config
    return st


@pytest.mark.parametrize("kw,t_init,status", [
    (dict(order=2, dims=(6,), ranks=(2, 2)), 3, L.STR_E_ARG),                   # N >= 3
    (dict(), 0, L.STR_E_SHAPE),                                                 # t_init >= 1
    (dict(dims=(6, 0, 4)), 3, L.STR_E_SHAPE),                                   # I_n >= 1
    (dict(ranks=(2, 0, 2, 2)), 3, L.STR_E_ARG),                                 # R_n in [1, 16]
    (dict(ranks=(2, 17, 2, 2)), 3, L.STR_E_ARG),
    (dict(ranks=(2, 12, 12, 2)), 3, L.STR_E_ARG),                               # R_n R_{n+1} <= 128
    (dict(split_k=3), 3, L.STR_E_ARG),                                          # split in [0, N-2]
    (dict(ranks=(1, 12, 8, 12), split_k=1), 3, L.STR_E_ARG),                    # STR: R_{k+1} R_N <= 128
    (dict(dtype=7), 3, L.STR_E_ARG),
    (dict(variant=9), 3, L.STR_E_ARG),
    (dict(world=2, rank=2), 3, L.STR_E_ARG),                                    # rank < world
    (dict(world=4, dims=(6, 5, 4)), 3, L.STR_E_PRECOND),                        # I_1 % p == 0
    (dict(variant=L.STR_SAMPLE_UNIFORM, m=5), 3, L.STR_E_PRECOND),              # m >= max R_n R_{n+1}
    (dict(variant=L.STR_SAMPLE_KSRFT, m=5), 3, L.STR_E_PRECOND),
    (dict(variant=L.STR_SAMPLE_LEVERAGE, m=100, world=2), 3, L.STR_E_PRECOND),  # rSTR runs as replicas only
])
def test_str_init_rejects_invalid_configs(kw, t_init, status):
    cfg, keep = _cfg(**kw)
    assert _init(cfg, t_init) == status


def test_str_init_null_arguments():
    cfg, keep = _cfg()
    out = C.c_void_p()
    cores = (C.POINTER(C.c_double) * 4)()
    assert L.lib.str_init(None, FAKE, 3, cores, C.byref(out)) == L.STR_E_ARG
    assert L.lib.str_init(C.byref(cfg), None, 3, cores, C.byref(out)) == L.STR_E_ARG
    assert L.lib.str_init(C.byref(cfg), FAKE, 3, None, C.byref(out)) == L.STR_E_ARG
    assert L.lib.str_init(C.byref(cfg), FAKE, 3, cores, None) == L.STR_E_ARG


def test_null_handle_everywhere():
    lib = L.lib
    buf = (C.c_double * 4)()
    idx = (C.c_int32 * 4)()
    a, b = C.c_double(), C.c_int64()
    assert lib.str_update_batch(None, FAKE, 1) == L.STR_E_ARG
    assert lib.str_update_batch_host(None, FAKE, 1) == L.STR_E_ARG
    assert lib.str_get_cores(None, 1, buf, 4) == L.STR_E_ARG
    assert lib.str_get_temporal_rows(None, 0, 1, buf) == L.STR_E_ARG
    assert lib.str_fit(None, FAKE, 0, 1, C.byref(a)) == L.STR_E_ARG
    assert lib.str_tr_als(None, FAKE, 1, 1, C.byref(a)) == L.STR_E_ARG
    assert lib.str_sync(None) == L.STR_E_ARG
    assert lib.str_set_profiling(None, 1) == L.STR_E_ARG
    assert lib.str_profile(None, C.byref(a), C.byref(b), C.byref(a), C.byref(b)) == L.STR_E_ARG
    assert lib.str_get_index_table(None, 1, idx, 4) == L.STR_E_ARG
    assert lib.str_set_index_table(None, 1, idx, 4) == L.STR_E_ARG
    assert lib.str_processed(None) == 0
    assert lib.str_kernel_launches(None) == 0
    assert lib.str_error_string(None) == b"null handle"
    lib.str_destroy(None)   # idempotent on NULL
