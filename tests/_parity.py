"""Shared helpers for GPU-vs-oracle parity runs (imported by the -m gpu tests only).

Metrics, all against the fp64 oracle:
  rel          per-core relative Frobenius error (temporal core included)
  row_rel      per-row maximum relative error of G_n(2): max_i ||g_i - o_i|| / max(||o_i||, 1e-3 rms_i ||o_i||)
               (a localized error in a few rows is not diluted by the norm)
  recon_rel    gauge-invariant ||X^_gpu - X^_oracle|| / ||X^_oracle|| over the temporal rows of the
               latest batch, X^_[N] = G_N(2) G^{≠N}_[2]^T (Eq. tr_als, n = N) evaluated by the
               oracle's own subchain, block by block over the last chain index.
"""
import numpy as np

from oracle.fit import relative_error
from oracle.stream import StreamingTR
from oracle.tralg import core_unfold, subchain, unfold2
from workloads import make_stream
from workloads.gen import paper_view


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def row_rel(a, b):
    """Per-row max relative error of the mode-2 unfoldings (rows = i_n) of two cores."""
    A, B = core_unfold(a), core_unfold(b)
    nb = np.linalg.norm(B, axis=1)
    floor = 1e-3 * float(np.sqrt(np.mean(nb ** 2))) if nb.size else 1.0
    return float(np.max(np.linalg.norm(A - B, axis=1) / np.maximum(nb, floor)))


def recon_rel(cores_a, cores_b, t0, t1):
    """||X^_a - X^_b|| / ||X^_b|| over temporal rows [t0, t1) (both core lists in paper layout)."""
    N = len(cores_a)
    ga = core_unfold(cores_a[-1][:, t0:t1, :])
    gb = core_unfold(cores_b[-1][:, t0:t1, :])
    d2 = n2 = 0.0
    I_last = cores_a[N - 2].shape[1]
    for i in range(I_last):
        Sa = unfold2(subchain(cores_a, N, last_index=i))
        Sb = unfold2(subchain(cores_b, N, last_index=i))
        xa = ga @ Sa.T
        xb = gb @ Sb.T
        d2 += float(np.sum((xa - xb) ** 2))
        n2 += float(np.sum(xb ** 2))
    return float(np.sqrt(d2 / n2)) if n2 > 0 else 0.0


def gpu_stream(name_or_cfg, contract=None, n_batches=None, fit_every=True, split_k=None, check=None, init=None):
    """Run oracle (fp64 CPU) and libstr (GPU) side by side on the same seeded stream.

    Yields (batch, per-core relative errors, oracle fit, gpu fit, handle, oracle) after init (batch -1)
    and after every update.  init: initial cores (default: the stream's perturbed-truth cores)."""
    import torch
    import paper_2307_00719_b200 as lib
    s = make_stream(name_or_cfg)
    cfg = s.cfg
    contract = contract or cfg.contract
    nb = cfg.n_batches if n_batches is None else n_batches
    Xi = s.init_slab()
    init = s.init_cores() if init is None else init
    orc = StreamingTR(paper_view(Xi), init)
    Xi_d = torch.from_numpy(Xi).to("cuda")
    h = lib.str_init(cfg.N, cfg.dims, cfg.ranks, Xi_d, cfg.t_init, init, dtype=cfg.dtype, contract=contract,
                     split_k=cfg.split_k if split_k is None else split_k)
    hist_np = [Xi]
    hist_d = [Xi_d]
    for b in range(-1, nb):
        if b >= 0:
            Xb = s.batch(b)
            Xb_d = torch.from_numpy(Xb).to("cuda")
            lib.str_update_batch(h, Xb_d, cfg.t_new)
            orc.update(paper_view(Xb))
            hist_np.append(Xb)
            hist_d.append(Xb_d)
        errs = [rel(lib.str_get_cores(h, n), orc.cores[n - 1]) for n in range(1, cfg.N + 1)]
        fo = fg = None
        if fit_every or b == nb - 1:
            Xall = np.concatenate(hist_np, axis=0)
            fo = relative_error(paper_view(Xall), orc.cores)
            fg = lib.str_fit(h, torch.cat(hist_d, dim=0), 0, lib.str_processed(h))
        yield b, errs, fo, fg, h, orc
