"""paper_2307_00719_b200 — B200-native streaming tensor-ring (STR / rSTR) per-batch update.

Thin Python binding over the C ABI in ``include/str.h`` (``libstr.so``, hand-written sm_100a
CUDA).  The functions below have the same names as the C entry points and only marshal
arguments: every step of the method runs in the library's kernels.  PyTorch is used only to
hold device memory and to name the CUDA stream.

Tensor data (X_init, X_new, fit slabs) are contiguous CUDA tensors holding the paper's
linearization (first index fastest) — e.g. a torch tensor of shape
(t, I_{N-1}, ..., I_1) in C order.  Cores are exchanged in the paper layout
(R_n, I_n, R_{n+1}) as fp64 numpy arrays.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (STR_CONTRACT_3XTF32, STR_CONTRACT_F64, STR_DET, STR_F32, STR_F64, STR_SAMPLE_KSRFT,
                   STR_SAMPLE_LEVERAGE, STR_SAMPLE_UNIFORM, StrError, str_config)

__all__ = ["str_init", "str_update_batch", "str_update_batch_host", "str_get_cores", "str_get_temporal_rows",
           "str_fit", "str_sync", "str_processed", "str_error_string", "str_destroy", "str_kernel_launches",
           "str_set_profiling", "str_profile", "str_get_index_table", "str_set_index_table", "str_tr_als", "Handle",
           "str_loopback_create", "str_loopback_destroy",
           "StrError",
           "LIB_PATH"]

LIB_PATH = _lib.LIB_PATH
_VARIANTS = {"det": STR_DET, "uniform": STR_SAMPLE_UNIFORM, "leverage": STR_SAMPLE_LEVERAGE, "ksrft": STR_SAMPLE_KSRFT}
_CONTRACTS = {"3xtf32": STR_CONTRACT_3XTF32, "f64": STR_CONTRACT_F64}
_DTYPES = {"f32": STR_F32, "f64": STR_F64}


class Handle:
    """Owns a ``str_state*``, the host-side config arrays it was created from and the CUDA stream
    the library enqueues on (a torch stream object, so that device buffers handed to the library
    can be recorded on it: the caching allocator then keeps them alive until the enqueued work
    that reads them has finished — include/str.h's lifetime rule for X)."""

    def __init__(self, ptr, N, dims, ranks, dtype, keep, stream=None):
        self.ptr = ptr
        self.N = N
        self.dims = tuple(dims)
        self.ranks = tuple(ranks)
        self.dtype = dtype
        self._keep = keep
        self.stream = stream

    def __del__(self):
        try:
            str_destroy(self)
        except Exception:
            pass


def _check(h: Optional[Handle], status: int):
    if status != 0:
        msg = _lib.lib.str_error_string(h.ptr).decode() if (h is not None and h.ptr) else ""
        raise StrError(status, msg)


def _dev_ptr(x, expect_numel: int, dtype: str) -> int:
    import torch
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError("expected a CUDA torch.Tensor (device pointer argument)")
    want = torch.float32 if dtype == "f32" else torch.float64
    if x.dtype != want or not x.is_contiguous():
        raise TypeError(f"expected a contiguous {want} tensor, got {x.dtype}")
    if x.numel() != expect_numel:
        raise ValueError(f"expected {expect_numel} elements, got {x.numel()}")
    return x.data_ptr()


def _enter(h: Optional[Handle], x, stream=None):
    """Orders the library stream after the caller's current stream (which produced x) and records
    x on the library stream (argument marshalling only: no data is touched)."""
    import torch
    st = stream if stream is not None else h.stream
    if st is None:
        return
    cur = torch.cuda.current_stream(x.device)
    if cur.cuda_stream != st.cuda_stream:
        st.wait_stream(cur)
    x.record_stream(st)


def str_init(order: int, dims: Sequence[int], ranks: Sequence[int], X_init, t_init: int,
             init_cores: Sequence[np.ndarray], *, dtype: str = "f32", contract: str = "3xtf32",
             variant: str = "det", sketch_rows: int = 0, seed: int = 0, t_capacity: int = 0, split_k: int = 0,
             world_size: int = 1, rank: int = 0, nccl_id: Optional[bytes] = None, device: int = 0,
             stream: Optional[int] = None, loopback_group: Optional[int] = None) -> Handle:
    """Alg. 4 l.1-5 / Alg. 7-8 init.  ``dims`` are the GLOBAL I_1..I_{N-1}; X_init is this rank's
    shard; ``init_cores`` are global paper-layout cores (core N has t_init rows)."""
    import torch
    N = int(order)
    dims_a = (C.c_int64 * (N - 1))(*[int(d) for d in dims])
    ranks_a = (C.c_int32 * N)(*[int(r) for r in ranks])
    # the library's stream: the caller's (wrapped so buffers can be recorded on it) or a dedicated
    # stream of this handle
    tstream = (torch.cuda.Stream(device) if not stream else torch.cuda.ExternalStream(int(stream), device=device))
    stream = tstream.cuda_stream
    nid = None
    if nccl_id is not None:
        nid = C.create_string_buffer(bytes(nccl_id), len(nccl_id))
    comm = _lib.STR_COMM_NCCL
    gptr = None
    if loopback_group is not None:   # in-process ranks sharing one GPU (str_loopback_create)
        comm = _lib.STR_COMM_LOOPBACK
        gptr = C.c_void_p(int(loopback_group))
    cfg = str_config(order=N, dims=dims_a, ranks=ranks_a, dtype=_DTYPES[dtype], contract=_CONTRACTS[contract],
                     variant=_VARIANTS[variant], sketch_rows=int(sketch_rows), seed=int(seed) & (2 ** 64 - 1),
                     t_capacity=int(t_capacity), split_k=int(split_k), world_size=int(world_size), rank=int(rank),
                     nccl_id=(gptr if gptr is not None else (C.cast(nid, C.c_void_p) if nid is not None else None)),
                     device=int(device), stream=C.c_void_p(stream), comm=comm)
    local = [int(d) for d in dims]
    local[0] //= int(world_size)
    xptr = _dev_ptr(X_init, int(np.prod(local)) * int(t_init), dtype)
    _enter(None, X_init, tstream)
    cores = [np.ascontiguousarray(np.asarray(G, dtype=np.float64).reshape(-1, order="F")) for G in init_cores]
    arr = (C.POINTER(C.c_double) * N)(*[c.ctypes.data_as(C.POINTER(C.c_double)) for c in cores])
    out = C.c_void_p()
    st = _lib.lib.str_init(C.byref(cfg), C.c_void_p(xptr), int(t_init), arr, C.byref(out))
    h = Handle(out, N, dims, ranks, dtype, keep=(dims_a, ranks_a, nid), stream=tstream)
    if st != 0:
        msg = _lib.lib.str_error_string(out).decode() if out.value else ""
        if out.value:
            _lib.lib.str_destroy(out)
            h.ptr = None
        raise StrError(st, msg)
    h.world_size = int(world_size)
    h.local_slice = int(np.prod(local))
    return h


def str_loopback_create(world_size: int) -> int:
    """In-process loopback group of world_size ranks (include/str.h): returns the group pointer."""
    g = C.c_void_p()
    _check(None, _lib.lib.str_loopback_create(int(world_size), C.byref(g)))
    return int(g.value)


def str_loopback_destroy(group: int) -> None:
    _lib.lib.str_loopback_destroy(C.c_void_p(int(group)))


def str_update_batch(h: Handle, X_new, t_new: Optional[int] = None) -> None:
    """One STR / rSTR step on a device-resident batch (Alg. 4 l.7-19)."""
    if t_new is None:
        t_new = X_new.numel() // h.local_slice
    ptr = _dev_ptr(X_new, h.local_slice * int(t_new), h.dtype)
    _enter(h, X_new)
    _check(h, _lib.lib.str_update_batch(h.ptr, C.c_void_p(ptr), int(t_new)))


def str_update_batch_host(h: Handle, X_host, t_new: int) -> None:
    """Same step with X_new in host memory (numpy array or pinned CPU tensor)."""
    if hasattr(X_host, "data_ptr"):
        ptr = X_host.data_ptr()
        n = X_host.numel()
    else:
        ptr = X_host.ctypes.data
        n = X_host.size
    if n != h.local_slice * int(t_new):
        raise ValueError("X_new size mismatch")
    _check(h, _lib.lib.str_update_batch_host(h.ptr, C.c_void_p(ptr), int(t_new)))


def str_get_cores(h: Handle, n: int) -> np.ndarray:
    """Global core n (1..N) in paper layout, shape (R_n, I_n, R_{n+1})."""
    N = h.N
    Rn, Rn1 = h.ranks[n - 1], h.ranks[n % N]
    I = str_processed(h) if n == N else h.dims[n - 1]
    out = np.empty(Rn * I * Rn1, dtype=np.float64)
    _check(h, _lib.lib.str_get_cores(h.ptr, int(n), out.ctypes.data_as(C.POINTER(C.c_double)), out.size))
    return out.reshape((Rn, I, Rn1), order="F")


def str_get_temporal_rows(h: Handle, t0: int, t: int) -> np.ndarray:
    """Rows [t0, t0+t) of G_N(2), shape (t, R_N R_1), column r_N + R_N r_1."""
    S = h.ranks[-1] * h.ranks[0]
    out = np.empty(int(t) * S, dtype=np.float64)
    _check(h, _lib.lib.str_get_temporal_rows(h.ptr, int(t0), int(t), out.ctypes.data_as(C.POINTER(C.c_double))))
    return out.reshape(int(t), S)


def str_fit(h: Handle, X, t0: int, t: int) -> float:
    ptr = _dev_ptr(X, h.local_slice * int(t), h.dtype)
    _enter(h, X)
    v = C.c_double()
    _check(h, _lib.lib.str_fit(h.ptr, C.c_void_p(ptr), int(t0), int(t), C.byref(v)))
    return v.value


def str_tr_als(h: Handle, X, t: int, sweeps: int) -> float:
    """Batch TR-ALS on the GPU (Alg. 1): `sweeps` sweeps in mode order N, 1..N-1 from the cores the
    handle holds, then the streaming state rebuilt from X (device, t slices).  Returns the fit
    ||X - TR(G)|| / ||X|| after the last sweep."""
    ptr = _dev_ptr(X, h.local_slice * int(t), h.dtype)
    _enter(h, X)
    v = C.c_double()
    _check(h, _lib.lib.str_tr_als(h.ptr, C.c_void_p(ptr), int(t), int(sweeps), C.byref(v)))
    return v.value


def str_sync(h: Handle) -> None:
    _check(h, _lib.lib.str_sync(h.ptr))


def str_processed(h: Handle) -> int:
    return int(_lib.lib.str_processed(h.ptr))


def str_error_string(h: Handle) -> str:
    return _lib.lib.str_error_string(h.ptr).decode()


def str_destroy(h: Handle) -> None:
    if h is not None and h.ptr:
        _lib.lib.str_destroy(h.ptr)
        h.ptr = None


def str_kernel_launches(h: Handle) -> int:
    return int(_lib.lib.str_kernel_launches(h.ptr))


def str_set_profiling(h: Handle, enable: bool) -> None:
    _check(h, _lib.lib.str_set_profiling(h.ptr, int(bool(enable))))


def str_profile(h: Handle):
    """(pass1_ms, pass1_launches, pass2_ms, pass2_launches) accumulated since profiling was enabled."""
    a, b = C.c_double(), C.c_double()
    na, nb = C.c_int64(), C.c_int64()
    _check(h, _lib.lib.str_profile(h.ptr, C.byref(a), C.byref(na), C.byref(b), C.byref(nb)))
    return a.value, na.value, b.value, nb.value


def str_get_index_table(h: Handle, mode: int, m: int) -> np.ndarray:
    out = np.empty(int(m), dtype=np.int32)
    _check(h, _lib.lib.str_get_index_table(h.ptr, int(mode), out.ctypes.data_as(C.POINTER(C.c_int32)), int(m)))
    return out


def str_set_index_table(h: Handle, mode: int, idx) -> None:
    a = np.ascontiguousarray(idx, dtype=np.int32)
    _check(h, _lib.lib.str_set_index_table(h.ptr, int(mode), a.ctypes.data_as(C.POINTER(C.c_int32)), a.size))
