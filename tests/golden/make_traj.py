"""Writes the cached oracle trajectories under tests/golden/traj/ (test fixtures).

Imports nothing but ``oracle/`` and ``workloads/``: every stored value is computed by the fp64
CPU oracle from the seeded synthetic inputs, never by the CUDA path.  The GPU parity tests
(tests/test_gpu_traj.py) load these files instead of re-running the oracle at full size, where
one oracle step costs seconds (C5: 20.5M entries per batch).

Files (numpy .npz, fp64):
  <cfg>_als_init.npz   TR-ALS initialization on X_init (Alg. 1; protocol P:734, P:752:
                       tol 1e-8 on the change of the relative error, <= 100 sweeps, from
                       workloads.gen.als_start_cores): init cores core1..coreN, init error, sweeps.
  <cfg>_<init>_traj.npz  STR (Alg. 4) from the init cores (init = "als" or "pert", the
                       perturbed-truth cores of workloads.gen.Stream.init_cores) over every batch:
                       b<b>_core<n> (n < N) after batch b, b<b>_gnew (t_new x R_N x R_1 new temporal
                       rows, paper layout R_N x t_new x R_1), fit[b] over the whole stream so far,
                       condQ[b, n] = cond(Q_n) after batch b.

    python tests/golden/make_traj.py C5 [C3 ...] [--fit-every K]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle.als import tr_als  # noqa: E402
from oracle.fit import relative_error  # noqa: E402
from oracle.stream import StreamingTR  # noqa: E402
from workloads import make_stream  # noqa: E402
from workloads.gen import als_start_cores, paper_view  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "traj")


def als_init(name: str, force: bool = False):
    path = os.path.join(OUT, f"{name}_als_init.npz")
    if os.path.exists(path) and not force:
        d = np.load(path)
        n = sum(1 for k in d.files if k.startswith("core"))
        return [d[f"core{i}"] for i in range(1, n + 1)]
    s = make_stream(name)
    X = paper_view(s.init_slab()).astype(np.float64)
    t0 = time.time()
    cores, err, sweeps = tr_als(X, s.cfg.ranks, als_start_cores(s.cfg), tol=1e-8, max_sweeps=100)
    print(f"{name}: TR-ALS init error {err:.3e} after {sweeps} sweeps ({time.time() - t0:.1f} s)", flush=True)
    np.savez_compressed(path, err=err, sweeps=sweeps, **{f"core{i + 1}": c for i, c in enumerate(cores)})
    return cores


def trajectory(name: str, init: str, fit_every: int = 1):
    s = make_stream(name)
    cfg = s.cfg
    cores = als_init(name) if init == "als" else s.init_cores()
    Xi = s.init_slab()
    orc = StreamingTR(paper_view(Xi), cores)
    hist = [Xi]
    out = {}
    fits = np.full(cfg.n_batches, np.nan)
    cond = np.zeros((cfg.n_batches, cfg.N - 1))
    t0 = time.time()
    for b in range(cfg.n_batches):
        Xb = s.batch(b)
        orc.update(paper_view(Xb))
        hist.append(Xb)
        for n in range(1, cfg.N):
            out[f"b{b}_core{n}"] = orc.cores[n - 1]
            cond[b, n - 1] = np.linalg.cond(orc.Q[n - 1])
        out[f"b{b}_gnew"] = orc.last_GN_new
        if (b + 1) % fit_every == 0 or b == cfg.n_batches - 1:
            fits[b] = relative_error(paper_view(np.concatenate(hist, axis=0)), orc.cores)
        print(f"{name}/{init} batch {b}: fit {fits[b]:.6e}  max cond(Q) {cond[b].max():.3e}  "
              f"({time.time() - t0:.1f} s)", flush=True)
    np.savez_compressed(os.path.join(OUT, f"{name}_{init}_traj.npz"), fit=fits, condQ=cond, **out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--init", default="als", choices=["als", "pert"])
    ap.add_argument("--fit-every", type=int, default=1)
    ap.add_argument("--only-init", action="store_true")
    a = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    for nm in a.configs:
        if a.only_init:
            als_init(nm)
        else:
            trajectory(nm, a.init, a.fit_every)
