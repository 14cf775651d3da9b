#!/usr/bin/env python
"""§4 comparison workload on the GPU (protocol P:733-767, sweeps P:799-862).

For each synthetic exact-TR tensor (N(0,1) cores, R_true = R): TR-ALS on the first 20% of the
temporal slices (tolerance 1e-8 on the change of relative error, at most 100 sweeps, from random
N(0,1) cores) initializes every method; then t_new slices arrive per step and each method records
its processing time for the step (CUDA events, synchronized) and the relative error of its
decomposition over all data so far.  Methods: STR (Alg. 4), rSTR-U / rSTR-L (Alg. 7/8, m = 1000),
GPU TR-ALS Hot (warm start from the previous step's cores) and Cold (fresh N(0,1) cores every
step), both with the batch baselines' settings (tolerance 1e-10, at most 50 sweeps).  The
MATLAB baselines themselves and the real datasets are out of scope.

    python tools/compare_sweeps.py [--set order|length|slice|rank|all] [--quick] [--out FILE]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def workloads(which, quick):
    """(label, dims (I_1..I_{N-1}), I_N, t_new, R)."""
    out = []
    if which in ("order", "all"):   # fig:order P:806-821
        out += [("300^3", (300, 300), 300, 5, 5), ("500^3", (500, 500), 500, 5, 5),
                ("40^5", (40, 40, 40, 40), 40, 5, 5), ("60^5", (60, 60, 60, 60), 60, 5, 5)]
    if which in ("length", "all"):  # fig:length P:823-832
        out += [(f"30^4x{n}", (30, 30, 30, 30), n, 5, 5) for n in (120, 160, 200)]
    if which in ("slice", "all"):   # fig:slice P:834-844
        out += [(f"30^4x200 t_new={t}", (30, 30, 30, 30), 200, t, 5) for t in (2, 6, 10)]
    if which in ("rank", "all"):    # fig:rank P:846-862
        out += [(f"30^4x200 R={r}", (30, 30, 30, 30), 200, 5, r) for r in (3, 4, 6)]
    if quick:
        out = [w for w in out if w[0] in ("300^3", "40^5", "30^4x120")] or out[:2]
    return out


def run_workload(label, dims, IN, t_new, R, methods, seed, max_steps, contract="3xtf32"):
    import torch
    import paper_2307_00719_b200 as lib
    from workloads.configs import StreamConfig
    from workloads import make_stream
    N = len(dims) + 1
    ranks = (R,) * N
    t_init = max(1, int(round(0.2 * IN)))
    n_batches = (IN - t_init) // t_new
    if max_steps:
        n_batches = min(n_batches, max_steps)
    cfg = StreamConfig(label, tuple(dims), ranks, t_init, t_new, n_batches, "f32", contract, core_scale=1.0,
                       noise_abs=0.0, seed=seed)
    s = make_stream(cfg)
    T_total = t_init + t_new * n_batches
    slice_n = int(np.prod(dims))
    # whole tensor on the device (the history the batch baselines re-read)
    hist = torch.empty(T_total * slice_n, dtype=torch.float32, device="cuda")
    hist[:t_init * slice_n] = torch.from_numpy(s.init_slab().reshape(-1)).cuda()
    for b in range(n_batches):
        a = (t_init + b * t_new) * slice_n
        hist[a:a + t_new * slice_n] = torch.from_numpy(s.batch(b).reshape(-1)).cuda()
    rng = np.random.default_rng(seed + 7)

    def rand_cores(tn):
        return [rng.standard_normal((R, dims[n] if n < N - 1 else tn, R)) for n in range(N)]

    def ev_time(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), r

    def als_to_convergence(h, T, tol, itmax):
        prev, err, it = None, None, 0
        for it in range(1, itmax + 1):
            err = lib.str_tr_als(h, hist[:T * slice_n], T, 1)
            if prev is not None and abs(prev - err) < tol:
                break
            prev = err
        return err, it

    # ---- initialization: TR-ALS on the first 20% (tol 1e-8, IT 100)
    h0 = lib.str_init(N, dims, ranks, hist[:t_init * slice_n], t_init, rand_cores(t_init), dtype="f32",
                      contract=contract)
    init_ms, (init_err, init_it) = ev_time(lambda: als_to_convergence(h0, t_init, 1e-8, 100))
    init_cores = [lib.str_get_cores(h0, n) for n in range(1, N + 1)]
    lib.str_destroy(h0)
    res = {"workload": label, "dims": list(dims), "I_N": IN, "t_init": t_init, "t_new": t_new, "R": R,
           "steps": n_batches, "init": {"ms": round(init_ms, 2), "sweeps": init_it, "rel_err": init_err},
           "methods": {}}
    for meth in methods:
        kw = {}
        if meth in ("rSTR-U", "rSTR-L", "rSTR-K"):
            kw = dict(variant={"rSTR-U": "uniform", "rSTR-L": "leverage", "rSTR-K": "ksrft"}[meth], sketch_rows=1000,
                      seed=seed)
        h = lib.str_init(N, dims, ranks, hist[:t_init * slice_n], t_init, init_cores, dtype="f32", contract=contract,
                         t_capacity=T_total + 8, **kw)
        times, errs = [], []
        T = t_init
        hc = None
        for b in range(n_batches):
            a = T * slice_n
            T += t_new
            if meth in ("STR", "rSTR-U", "rSTR-L", "rSTR-K"):
                ms, _ = ev_time(lambda: (lib.str_update_batch(h, hist[a:a + t_new * slice_n], t_new),
                                         lib.str_sync(h)))
                err = lib.str_fit(h, hist[:T * slice_n], 0, T)
            elif meth == "TR-ALS Hot":   # warm start: previous cores, new temporal rows from one STR solve
                def hot():
                    lib.str_update_batch(h, hist[a:a + t_new * slice_n], t_new)
                    return als_to_convergence(h, T, 1e-10, 50)
                ms, (err, _) = ev_time(hot)
            else:                         # TR-ALS Cold: fresh random cores every step
                if hc is not None:
                    lib.str_destroy(hc)
                hc = lib.str_init(N, dims, ranks, hist[:T * slice_n], T, rand_cores(T), dtype="f32", contract=contract)
                ms, (err, _) = ev_time(lambda: als_to_convergence(hc, T, 1e-10, 50))
            times.append(ms)
            errs.append(err)
        if hc is not None:
            lib.str_destroy(hc)
        lib.str_destroy(h)
        res["methods"][meth] = {"ms_per_step_mean": round(float(np.mean(times)), 4),
                                "ms_per_step_median": round(float(np.median(times)), 4),
                                "total_ms": round(float(np.sum(times)), 2),
                                "rel_err_final": errs[-1], "rel_err_max": float(np.max(errs)),
                                "ms_series": [round(t, 4) for t in times], "err_series": errs}
    del hist
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", default="order", choices=["order", "length", "slice", "rank", "all"])
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--methods", default="STR,rSTR-U,rSTR-L,rSTR-K,TR-ALS Hot,TR-ALS Cold")
    ap.add_argument("--max-steps", type=int, default=0)
    ap.add_argument("--seed", type=int, default=2307)
    ap.add_argument("--contract", default="3xtf32", choices=["3xtf32", "f64"])
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "compare.json"))
    a = ap.parse_args()
    methods = [m.strip() for m in a.methods.split(",")]
    results = []
    for (label, dims, IN, t_new, R) in workloads(a.set, a.quick):
        t = time.time()
        r = run_workload(label, dims, IN, t_new, R, methods, a.seed, a.max_steps, a.contract)
        r["contract"] = a.contract
        r["wall_s"] = round(time.time() - t, 1)
        results.append(r)
        line = " | ".join(f"{m}: {v['ms_per_step_mean']:.3f} ms, err {v['rel_err_final']:.2e}"
                          for m, v in r["methods"].items())
        print(f"{label} ({r['steps']} steps, init {r['init']['sweeps']} sweeps err {r['init']['rel_err']:.1e}): {line}",
              flush=True)
        json.dump(results, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
