"""ctypes binding of include/str.h — argument marshalling only.

Every step of the update runs inside libstr.so (sm_100a CUDA kernels).  There is no Python or
CPU fallback: if the shared library is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libstr.so")

STR_OK, STR_E_ARG, STR_E_SHAPE, STR_E_PRECOND, STR_E_NUMERIC, STR_E_CUDA, STR_E_NCCL, STR_E_OOM, STR_E_POISONED = range(9)
STATUS_NAMES = ["STR_OK", "STR_E_ARG", "STR_E_SHAPE", "STR_E_PRECOND", "STR_E_NUMERIC", "STR_E_CUDA", "STR_E_NCCL",
                "STR_E_OOM", "STR_E_POISONED"]
STR_F32, STR_F64 = 0, 1
STR_CONTRACT_3XTF32, STR_CONTRACT_F64 = 0, 1
STR_DET, STR_SAMPLE_UNIFORM, STR_SAMPLE_LEVERAGE, STR_SAMPLE_KSRFT = 0, 1, 2, 3
STR_COMM_NCCL, STR_COMM_LOOPBACK = 0, 1

# Every symbol include/str.h declares (checked by tests/test_abi.py without a GPU).
EXPORTS = ["str_init", "str_update_batch", "str_update_batch_host", "str_get_cores", "str_get_temporal_rows",
           "str_fit", "str_sync", "str_processed", "str_error_string", "str_destroy", "str_kernel_launches",
           "str_set_profiling", "str_profile", "str_get_index_table", "str_set_index_table", "str_tr_als",
           "str_loopback_create", "str_loopback_destroy"]


class str_config(C.Structure):
    _fields_ = [
        ("order", C.c_int32),
        ("dims", C.POINTER(C.c_int64)),
        ("ranks", C.POINTER(C.c_int32)),
        ("dtype", C.c_int),
        ("contract", C.c_int),
        ("variant", C.c_int),
        ("sketch_rows", C.c_int64),
        ("seed", C.c_uint64),
        ("t_capacity", C.c_int64),
        ("split_k", C.c_int32),
        ("world_size", C.c_int32),
        ("rank", C.c_int32),
        ("nccl_id", C.c_void_p),
        ("device", C.c_int32),
        ("stream", C.c_void_p),
        ("comm", C.c_int32),
    ]


class StrError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{name}: {msg}")


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found — build it with `python paper_2307_00719_b200/build.py` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    sig = {
        "str_init": (C.c_int, [C.POINTER(str_config), P, C.c_int64, C.POINTER(C.POINTER(C.c_double)),
                               C.POINTER(P)]),
        "str_update_batch": (C.c_int, [P, P, C.c_int64]),
        "str_update_batch_host": (C.c_int, [P, P, C.c_int64]),
        "str_get_cores": (C.c_int, [P, C.c_int32, C.POINTER(C.c_double), C.c_int64]),
        "str_get_temporal_rows": (C.c_int, [P, C.c_int64, C.c_int64, C.POINTER(C.c_double)]),
        "str_fit": (C.c_int, [P, P, C.c_int64, C.c_int64, C.POINTER(C.c_double)]),
        "str_tr_als": (C.c_int, [P, P, C.c_int64, C.c_int32, C.POINTER(C.c_double)]),
        "str_sync": (C.c_int, [P]),
        "str_processed": (C.c_int64, [P]),
        "str_error_string": (C.c_char_p, [P]),
        "str_destroy": (None, [P]),
        "str_kernel_launches": (C.c_int64, [P]),
        "str_set_profiling": (C.c_int, [P, C.c_int32]),
        "str_profile": (C.c_int, [P, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                  C.POINTER(C.c_int64)]),
        "str_get_index_table": (C.c_int, [P, C.c_int32, C.POINTER(C.c_int32), C.c_int64]),
        "str_set_index_table": (C.c_int, [P, C.c_int32, C.POINTER(C.c_int32), C.c_int64]),
        "str_loopback_create": (C.c_int, [C.c_int32, C.POINTER(P)]),
        "str_loopback_destroy": (None, [P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()
