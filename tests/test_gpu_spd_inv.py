"""Unit test of the library's SPD inverse (the "^{-1}" of G_n(2) = P_n Q_n^{-1}, Alg. 4 l.17 P:379:
a block Cholesky factor V = L^{-1} of sym(Q), Q^{-1} = V^T V; one CTA for S <= 32, a two-CTA cluster
above) against LAPACK on random SPD matrices of every size class (ragged S, one pivot block, both
kernel paths, the 128 maximum) and condition numbers up to 1e8; a non-SPD matrix must raise the
pivot-failure flag."""
import ctypes as C

import numpy as np
import pytest


def _inv(Qs):
    import paper_2307_00719_b200 as lib
    L = lib._lib.lib
    f = L.strdbg_spd_inv
    f.restype = C.c_int
    f.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.POINTER(C.c_int32), C.c_int32,
                  C.POINTER(C.c_float)]
    Qs = np.ascontiguousarray(np.stack(Qs), dtype=np.float64)
    out = np.empty_like(Qs)
    info = C.c_int32(0)
    st = f(0, Qs.shape[1], Qs.shape[0], Qs.ctypes.data, out.ctypes.data, C.byref(info), 0, None)
    assert st == 0
    return out, info.value


def _spd(S, cond, rng):
    U, _ = np.linalg.qr(rng.standard_normal((S, S)))
    w = np.logspace(0, np.log10(cond), S)
    rng.shuffle(w)
    return (U * w) @ U.T


@pytest.mark.gpu
@pytest.mark.parametrize("S", [1, 3, 8, 9, 15, 25, 64, 99, 100, 120, 128])
@pytest.mark.parametrize("cond", [1e1, 1e4, 1e8])
def test_spd_inverse_matches_lapack(S, cond):
    rng = np.random.default_rng(S * 7 + int(np.log10(cond)))
    Qs = [_spd(S, cond, rng) for _ in range(3)]
    # an unsymmetrized input: an antisymmetric part that the library's (Q + Q^T)/2 (reading R5) removes
    A = rng.standard_normal((S, S)) * 1e-3 * np.abs(Qs[2]).max()
    Qs[2] = Qs[2] + (A - A.T)
    out, info = _inv(Qs)
    assert info == 0
    for Q, Qi in zip(Qs, out):
        ref = np.linalg.inv(0.5 * (Q + Q.T))
        err = np.linalg.norm(Qi - ref) / np.linalg.norm(ref)
        # backward-stable SPD inversion: error ~ cond * eps
        assert err <= max(1e-13, 50 * cond * np.finfo(float).eps), (S, cond, err)
        assert np.linalg.norm(Qi - Qi.T) <= max(1e-13, 50 * cond * np.finfo(float).eps) * np.linalg.norm(ref)


@pytest.mark.gpu
def test_spd_inverse_flags_indefinite():
    rng = np.random.default_rng(3)
    Q = _spd(40, 10.0, rng)
    Q[17, 17] = -5.0
    _, info = _inv([Q])
    assert info == 1
