"""Seeded stream generator.

Every random draw uses ``numpy.random.Generator(PCG64(SeedSequence([seed, purpose, index])))``
so a temporal slice is the same whatever the batching.  Purposes:

  1 = true non-temporal core n, 2 = true temporal slice t, 3 = noise of slice t,
  4 = init perturbation of core n, 5 = init perturbation of temporal slice t,
  6 = video blob parameters.

Layout: a slab of ``t`` temporal slices is returned as a C-contiguous array of shape
``(t, I_{N-1}, ..., I_1)``, i.e. the paper's linearization with the first index fastest
(PAPER.md P:119).  ``paper_view`` gives the same memory as shape ``(I_1, ..., I_{N-1}, t)``.

The TR data are formed here with plain numpy products of this module's own cores; this is
input synthesis, not an implementation of any step of STR (the oracle and the CUDA path
each implement the method independently).
"""
from __future__ import annotations

from typing import List

import numpy as np

from .configs import StreamConfig, get_config

P_CORE, P_TSLICE, P_NOISE, P_INIT_CORE, P_INIT_T, P_VIDEO = 1, 2, 3, 4, 5, 6


def _rng(seed: int, purpose: int, index: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, purpose, index])))


def paper_view(slab: np.ndarray) -> np.ndarray:
    """(t, I_{N-1}, ..., I_1) C-order  ->  (I_1, ..., I_{N-1}, t) view of the same memory."""
    return slab.transpose(tuple(range(slab.ndim - 1, -1, -1)))


class Stream:
    """One synthetic stream: true cores (for 'tr' data), slabs, init cores."""

    def __init__(self, cfg: StreamConfig):
        self.cfg = cfg
        N, R = cfg.N, cfg.ranks
        self.np_dtype = np.float64 if cfg.dtype == "f64" else np.float32
        if cfg.kind == "tr":
            # True core n (1-based n = 1..N-1): paper layout (R_n, I_n, R_{n+1}).
            self.cores = []
            for n in range(1, N):
                Rn, Rn1 = R[n - 1], R[n % N]
                g = _rng(cfg.seed, P_CORE, n).standard_normal((Rn, cfg.dims[n - 1], Rn1))
                self.cores.append(g * cfg.core_scale)
            self._prep_tables()
        elif cfg.kind == "video":
            self._prep_video()
        else:
            raise ValueError(cfg.kind)

    # ---------------------------------------------------------------- true TR data
    def temporal_slice(self, t: int) -> np.ndarray:
        """True temporal slice g*_t (R_N x R_1)."""
        cfg = self.cfg
        if cfg.kind == "tr":
            RN, R1 = cfg.ranks[-1], cfg.ranks[0]
            return _rng(cfg.seed, P_TSLICE, t).standard_normal((RN, R1)) * cfg.core_scale
        a = 0.5 * (1.0 + np.sin(2 * np.pi * t / self.vP + self.vpsi))
        return np.diag(self.vw * a / self.vmax)

    def _slices(self, core: np.ndarray) -> np.ndarray:
        return np.ascontiguousarray(core.transpose(1, 0, 2))  # (I, R_n, R_{n+1})

    def _prep_tables(self):
        cfg = self.cfg
        N = cfg.N
        self._kg = max(1, (N - 1) // 2)
        # Left table over modes 1..kg, right table over modes kg+1..N-1 (first index fastest).
        A = self._slices(self.cores[0])
        for n in range(1, self._kg):
            S = self._slices(self.cores[n])
            A = np.einsum("xab,ybc->yxac", A, S).reshape(-1, A.shape[1], S.shape[2])
        B = self._slices(self.cores[self._kg])
        for n in range(self._kg + 1, N - 1):
            S = self._slices(self.cores[n])
            B = np.einsum("xab,ybc->yxac", B, S).reshape(-1, B.shape[1], S.shape[2])
        self._A = A                      # (L, R_1, R_{kg+1})
        self._B = B                      # (Rr, R_{kg+1}, R_N)

    def _clean_slice_tr(self, t: int) -> np.ndarray:
        g = self.temporal_slice(t)                                     # (R_N, R_1)
        C = np.einsum("rbc,ca->abr", self._B, g)                       # (R_1, R_kg+1, Rr)
        L = self._A.shape[0]
        X = self._A.reshape(L, -1) @ C.reshape(-1, C.shape[2])         # (L, Rr)
        return X.T                                                     # memory (r, l)

    # ---------------------------------------------------------------- video data (C3)
    def _prep_video(self):
        cfg = self.cfg
        H, W = cfg.dims
        K = cfg.ranks[0]
        r = _rng(cfg.seed, P_VIDEO, 0)
        cy = r.uniform(0, H, K)
        cx = r.uniform(0, W, K)
        sy = r.uniform(24, 80, K)
        sx = r.uniform(24, 80, K)
        self.vP = r.uniform(50, 300, K)
        self.vpsi = r.uniform(0, 2 * np.pi, K)
        self.vw = r.uniform(0.5, 1.0, K)
        y = np.arange(H)[:, None]
        x = np.arange(W)[:, None]
        self.vg = np.exp(-((y - cy) ** 2) / (2 * sy ** 2))  # (H, K)
        self.vh = np.exp(-((x - cx) ** 2) / (2 * sx ** 2))  # (W, K)
        # Global max over all frames, computed once (values then lie in [0, 1]).
        self.vmax = 1.0
        m = 0.0
        T = cfg.T_total
        for t0 in range(0, T, 64):
            ts = np.arange(t0, min(T, t0 + 64))
            a = 0.5 * (1.0 + np.sin(2 * np.pi * ts[:, None] / self.vP + self.vpsi))  # (t, K)
            Xc = np.einsum("hk,wk,tk->thw", self.vg, self.vh, a * self.vw)
            m = max(m, float(Xc.max()))
        self.vmax = m
        # Diagonal (CP) TR cores: G_1(y) = diag(g(y)), G_2(x) = diag(h(x)).
        self.cores = []
        for mat in (self.vg, self.vh):
            I = mat.shape[0]
            G = np.zeros((K, I, K))
            for k in range(K):
                G[k, :, k] = mat[:, k]
            self.cores.append(G)

    def _clean_slice_video(self, t: int) -> np.ndarray:
        a = 0.5 * (1.0 + np.sin(2 * np.pi * t / self.vP + self.vpsi)) * self.vw / self.vmax
        X = (self.vg * a) @ self.vh.T   # (H, W): memory index y + H x  -> C-order (W, H)
        return X.T

    # ---------------------------------------------------------------- slabs
    def slab(self, t0: int, t: int) -> np.ndarray:
        """Temporal slices [t0, t0+t) as C-order (t, I_{N-1}, ..., I_1) in the config dtype."""
        cfg = self.cfg
        shape_rev = tuple(reversed(cfg.dims))
        out = np.empty((t,) + shape_rev, dtype=self.np_dtype)
        for j in range(t):
            tt = t0 + j
            clean = self._clean_slice_tr(tt) if cfg.kind == "tr" else self._clean_slice_video(tt)
            clean = clean.reshape(shape_rev)
            if cfg.noise_abs > 0:
                clean = clean + cfg.noise_abs * _rng(cfg.seed, P_NOISE, tt).standard_normal(shape_rev)
            out[j] = clean
        return out

    def init_slab(self) -> np.ndarray:
        return self.slab(0, self.cfg.t_init)

    def batch(self, b: int) -> np.ndarray:
        """Batch b (0-based) of the update stream."""
        cfg = self.cfg
        return self.slab(cfg.t_init + b * cfg.t_new, cfg.t_new)

    # ---------------------------------------------------------------- init cores
    def init_cores(self) -> List[np.ndarray]:
        """Truth-based initial cores (Remark P:386-392 allows any feasible init).

        Non-temporal: true core + init_perturb * rms(core) * N(0,1).
        Temporal: true slices of the first t_init steps, perturbed the same way,
        in paper layout (R_N, t_init, R_1).
        """
        cfg = self.cfg
        out = []
        for n, G in enumerate(self.cores, start=1):
            s = float(np.sqrt(np.mean(G ** 2)))
            out.append(G + cfg.init_perturb * s * _rng(cfg.seed, P_INIT_CORE, n).standard_normal(G.shape))
        RN, R1 = cfg.ranks[-1], cfg.ranks[0]
        GN = np.empty((RN, cfg.t_init, R1))
        for t in range(cfg.t_init):
            g = self.temporal_slice(t)
            s = float(np.sqrt(np.mean(g ** 2))) or 1.0
            GN[:, t, :] = g + cfg.init_perturb * s * _rng(cfg.seed, P_INIT_T, t).standard_normal(g.shape)
        out.append(GN)
        return out


def make_stream(cfg) -> Stream:
    if isinstance(cfg, str):
        cfg = get_config(cfg)
    return Stream(cfg)


P_ALS_START = 7


def als_start_cores(cfg) -> List[np.ndarray]:
    """Random starting cores for batch TR-ALS on X_init (the initialization protocol of P:734,
    P:752): i.i.d. N(0, 1) entries scaled by 1/sqrt(R_n R_{n+1}), seeded
    by (seed, purpose 7, n); the temporal core has t_init rows.  Paper layout (R_n, I_n, R_{n+1})."""
    if isinstance(cfg, str):
        cfg = get_config(cfg)
    N, R = cfg.N, cfg.ranks
    sizes = list(cfg.dims) + [cfg.t_init]
    out = []
    for n in range(1, N + 1):
        Rn, Rn1 = R[n - 1], R[n % N]
        g = _rng(cfg.seed, P_ALS_START, n).standard_normal((Rn, sizes[n - 1], Rn1))
        out.append(g / np.sqrt(Rn * Rn1))
    return out
