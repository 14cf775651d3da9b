"""Shared helpers for GPU-vs-oracle parity runs (imported by the -m gpu tests only)."""
import numpy as np

from oracle.fit import relative_error
from oracle.stream import StreamingTR
from workloads import make_stream
from workloads.gen import paper_view


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def gpu_stream(name_or_cfg, contract=None, n_batches=None, fit_every=True, split_k=None, check=None):
    """Run oracle (fp64 CPU) and libstr (GPU) side by side on the same seeded stream.

    Yields (batch, per-core relative errors, oracle fit, gpu fit) after init (batch -1) and
    after every update."""
    import torch
    import paper_2307_00719_b200 as lib
    s = make_stream(name_or_cfg)
    cfg = s.cfg
    contract = contract or cfg.contract
    nb = cfg.n_batches if n_batches is None else n_batches
    Xi = s.init_slab()
    init = s.init_cores()
    orc = StreamingTR(paper_view(Xi), init)
    tdt = torch.float32 if cfg.dtype == "f32" else torch.float64
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
