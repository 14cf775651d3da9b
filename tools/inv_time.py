"""Isolated timing of the library's SPD inverse (strdbg_spd_inv, back-to-back launches)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_00719_b200 as lib  # noqa: E402

f = lib._lib.lib.strdbg_spd_inv
f.restype = C.c_int
f.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.POINTER(C.c_int32), C.c_int32,
              C.POINTER(C.c_float)]
rng = np.random.default_rng(0)
for S in (25, 64, 100, 128):
    A = rng.standard_normal((2 * S, S))
    Q = np.ascontiguousarray(A.T @ A)
    out = np.empty_like(Q)
    info = C.c_int32(0)
    us = C.c_float(0)
    f(0, S, 1, Q.ctypes.data, out.ctypes.data, C.byref(info), 200, C.byref(us))
    print(f"S={S}: {us.value:.2f} us per inverse (info {info.value}, err {np.abs(out @ Q - np.eye(S)).max():.1e})")
