#!/usr/bin/env python
"""STR update throughput on B200 (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]

A step is one ``str_update_batch`` — the whole per-batch STR update of Alg. 4:
temporal solve, every non-temporal P/Q accumulation and re-solve — on one batch X_new of
the workload (default C5: order-5 40^4 x t_new=8 fp32, TR ranks 10; BASELINE.json configs[4],
the configuration on which BASELINE.json quotes multi-GPU throughput).  X_new is sharded along
mode 1 across the N ranks (strong scaling: the global batch is fixed).  Inputs rotate through
15 distinct device-resident batches (1.2 GB > 126 MB L2), so no step reads an L2-warm batch.

Timing: W untimed warm-up steps, then K steps between CUDA events on the library's stream,
bracketed by a barrier + synchronize; the max over ranks is reported.  `e2e` repeats the
measurement through the public host-buffer API (pinned H2D of the shard + D2H of the new
temporal rows every step).  `roofline` times the dominant kernels (the two contraction
passes) with CUDA events on the library's stream.  `cpu_baseline` times the fp64 oracle
(test infrastructure, rank 0 only, bounded sample).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "STR update throughput (tensor entries ingested/s)"
UNIT = "entries/s"
N_DISTINCT = 15


def load_peaks():
    """MEASURED_PEAKS.json (driver-written: HBM copy, cuBLAS bf16) plus profiles/r02_measured_peaks.json
    (tools/measure_peaks.py on this pool's B200: cuBLAS TF32 and FP64 GEMM, burst and sustained)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks, src = json.load(f), "measured"
    except Exception:
        peaks, src = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"
    try:
        with open(os.path.join(ROOT, "profiles", "r02_measured_peaks.json")) as f:
            extra = json.load(f)
        peaks["tf32_tflops"] = extra["tf32"]["burst_tflops"]
        peaks["tf32_tflops_sustained"] = extra["tf32"]["sustained_tflops"]
        peaks["fp64_tflops"] = extra["fp64"]["burst_tflops"]
        peaks["fp64_tflops_sustained"] = extra["fp64"]["sustained_tflops"]
    except Exception:
        pass
    return peaks, src


def host_info():
    """CPU model, numpy version, BLAS vendor and its thread count (for the cpu_baseline record)."""
    import platform
    model = platform.processor() or "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    blas, threads = "unknown", os.cpu_count()
    try:
        from threadpoolctl import threadpool_info
        for d in threadpool_info():
            if d.get("user_api") == "blas":
                blas = f"{d.get('internal_api')} {d.get('version')} ({d.get('architecture')})"
                threads = d.get("num_threads", threads)
                break
    except Exception:
        pass
    return {"cpu_model": model, "numpy": np.__version__, "blas": blas, "blas_threads": threads,
            "host_cores": os.cpu_count()}


def nccl_summary(path_glob):
    """What NCCL_DEBUG=INFO said on this rank: version, NVLS use, transport lines (a few)."""
    import glob
    lines = []
    for fn in sorted(glob.glob(path_glob)):
        try:
            lines += open(fn).read().splitlines()
        except Exception:
            pass
    if not lines:
        return None
    ver = next((l.split("NCCL version", 1)[1].strip() for l in lines if "NCCL version" in l), None)
    nvls = [l for l in lines if "NVLS" in l]
    via = sorted({l.split("via", 1)[1].strip() for l in lines if " via " in l})[:4]
    return {"version": ver, "nvls_lines": len(nvls), "nvls_sample": nvls[:2], "transports": via,
            "lines": len(lines)}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}; launch with torchrun for N>1")
    return world, rank, local


def shard(slab: np.ndarray, world: int, rank: int) -> np.ndarray:
    I1 = slab.shape[-1]
    w = I1 // world
    return np.ascontiguousarray(slab[..., rank * w:(rank + 1) * w])


def bench_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2307_00719_b200 as lib
    from workloads import get_config, make_stream

    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl_glob = None
    if world > 1:
        # NCCL's own account of the collectives (NVLS / transports), summarised in the JSON line
        import tempfile
        ddir = os.environ.get("STR_NCCL_DEBUG_DIR") or tempfile.mkdtemp(prefix="str_nccl_")
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", os.path.join(ddir, "nccl.%h.%p.log"))
        nccl_glob = os.path.join(ddir, "nccl.*.log")
        dist.init_process_group("nccl", device_id=dev)
    cfg = get_config(args.config)
    if args.split_k is not None:   # two-pass split point override (tuning)
        cfg = cfg.with_(split_k=args.split_k)
    contract = args.contract or cfg.contract
    s = make_stream(cfg)
    # inputs: init slab + N_DISTINCT rotating batches, this rank's mode-1 shard, device-resident
    Xi = shard(s.init_slab(), world, rank)
    nd = min(N_DISTINCT, cfg.n_batches)
    host = [shard(s.batch(b), world, rank) for b in range(nd)]
    dev_batches = [torch.from_numpy(x).to(dev) for x in host]
    init = s.init_cores()
    nccl_id = None
    if world > 1:
        obj = [torch.cuda.nccl.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    stream = torch.cuda.Stream(dev)
    total_steps = args.warmup + args.steps
    cap = cfg.t_init + cfg.t_new * (2 * total_steps + 2 * args.e2e_steps + 64)
    with torch.cuda.stream(stream):
        vkw = {}
        if args.variant != "det":   # rSTR-U / -L / -K (Alg. 7 / 8 / 9) with the config's sketch size
            vkw = dict(variant=args.variant, sketch_rows=cfg.sketch_rows or 2000, seed=cfg.seed)
        h = lib.str_init(cfg.N, cfg.dims, cfg.ranks, torch.from_numpy(Xi).to(dev), cfg.t_init, init, dtype=cfg.dtype,
                         contract=contract, split_k=cfg.split_k, t_capacity=cap, world_size=world, rank=rank,
                         nccl_id=nccl_id, device=local, stream=stream.cuda_stream, **vkw)
    lib.str_sync(h)

    def barrier():
        if world > 1:
            dist.barrier()

    def maxall(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    step = [0]

    def one_step():
        lib.str_update_batch(h, dev_batches[step[0] % nd], cfg.t_new)
        step[0] += 1

    for _ in range(args.warmup):
        one_step()
    lib.str_sync(h)
    barrier()
    torch.cuda.synchronize(dev)
    l0 = lib.str_kernel_launches(h)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            one_step()
        e1.record(stream)
        lib.str_sync(h)
        torch.cuda.synchronize(dev)
    barrier()
    launches = lib.str_kernel_launches(h) - l0
    ms = maxall(e0.elapsed_time(e1))
    global_entries = cfg.batch_entries
    value = args.steps * global_entries / (ms / 1e3)

    # ---- per-batch latency: an event pair around each of K further steps (after
    # the timed region, so the throughput above carries no per-step events); median, p90 and the
    # trend against the processed length T (the step must not grow with the history)
    lat = []
    for _ in range(args.steps):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        one_step()
        a1.record(stream)
        lat.append((a0, a1))
    torch.cuda.synchronize(dev)
    lat_ms = np.array([maxall(a.elapsed_time(b)) for a, b in lat])
    slope = float(np.polyfit(np.arange(len(lat_ms)) * cfg.t_new, lat_ms * 1e3, 1)[0]) if len(lat_ms) > 2 else None
    latency = {"median_ms": round(float(np.median(lat_ms)), 5), "p90_ms": round(float(np.percentile(lat_ms, 90)), 5),
               "min_ms": round(float(lat_ms.min()), 5), "max_ms": round(float(lat_ms.max()), 5),
               "slope_us_per_slice": round(slope, 5) if slope is not None else None,
               "T_range": [int(lib.str_processed(h) - len(lat_ms) * cfg.t_new), int(lib.str_processed(h))],
               "note": "events around each step (adds the event overhead per step)"}

    # ---- roofline of the dominant kernels (contraction passes), events on the library stream;
    # the kernels also stamp %globaltimer per CTA (diagnostic trace) for their in-kernel span
    Ld = lib._lib.lib
    span = None
    if hasattr(Ld, "strdbg_tftrace") and contract == "3xtf32":
        Ld.strdbg_tftrace.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_longlong)]
        Ld.strdbg_tftrace(h.ptr, 1, None)
    lib.str_set_profiling(h, True)
    kp = min(args.steps, 10)
    for _ in range(kp):
        one_step()
    p1_ms, p1_n, p2_ms, p2_n = lib.str_profile(h)
    lib.str_set_profiling(h, False)
    if hasattr(Ld, "strdbg_tftrace") and contract == "3xtf32":
        Wd = 1024 + 4 * 160
        tr = np.zeros(2 * Wd, dtype=np.int64)
        Ld.strdbg_tftrace(h.ptr, 0, tr.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)))
        span = []
        for pas in (0, 1):
            g = tr[pas * Wd + 1024:(pas + 1) * Wd].reshape(160, 4)
            g = g[g[:, 0] > 0]
            span.append(float(g[:, 3].max() - g[:, 0].min()) / 1e3 if len(g) else None)
    peaks, peaks_src = load_peaks()
    R2 = cfg.ranks[0] * cfg.ranks[-1]
    local_entries = global_entries // world
    flops_per_pass = 2.0 * local_entries * R2          # algorithmic: 2 |X_new| R^2 per pass
    bytes_per_pass = local_entries * (4 if cfg.dtype == "f32" else 8)
    avg_p1 = p1_ms / max(p1_n, 1)
    avg_p2 = p2_ms / max(p2_n, 1)
    avg_pass = 0.5 * (avg_p1 + avg_p2)
    if contract == "3xtf32":
        # the pass kernels run inside a long, back-to-back step: the sustained TF32 figure (measured
        # cuBLAS TF32 GEMM), / 3 for the three TF32 MMAs per algorithmic multiply-add
        if "tf32_tflops_sustained" in peaks:
            peak_tf = peaks["tf32_tflops_sustained"] / 3.0
            basis = (f"measured cuBLAS TF32 GEMM sustained {peaks['tf32_tflops_sustained']} TF/s "
                     "(profiles/r02_measured_peaks.json) / 3 (3xTF32)")
            alt = {"tf32_burst": peaks["tf32_tflops"] / 3.0,
                   "bf16_burst_x_nominal_ratio": peaks["bf16_tflops"] * 0.5 / 3.0}
        else:
            peak_tf = peaks["bf16_tflops"] * 0.5 / 3.0   # nominal tf32/bf16 ratio (1.1 / 2.25 PF dense)
            basis = f"{peaks_src} bf16 burst {peaks['bf16_tflops']} x 0.5 (tf32/bf16 nominal) / 3 (3xTF32)"
            alt = {}
        bound, unit = "tensor", "TFLOP/s"
    else:
        # the FP64 path runs on the FP64 tensor cores (DMMA): measured cuBLAS DGEMM, sustained
        if "fp64_tflops_sustained" in peaks:
            peak_tf = peaks["fp64_tflops_sustained"]
            basis = f"measured cuBLAS FP64 GEMM sustained {peak_tf} TF/s (profiles/r02_measured_peaks.json)"
            alt = {"fp64_derived_clock_x_units": 148 * 64 * 2 * 1.965e9 / 1e12}
        else:
            peak_tf = 148 * 64 * 2 * 1.965e9 / 1e12       # FP64 FMA lanes x clock
            basis = "FP64: 148 SMs x 64 FMA/clk x 2 x 1.965 GHz"
            alt = {}
        bound, unit = "tensor", "TFLOP/s"
    if avg_pass <= 0:   # rSTR: no dense contraction pass on the path (sampled GEMMs only)
        avg_pass = float("nan")
    achieved = flops_per_pass / (avg_pass / 1e3) / 1e12
    t_hbm = bytes_per_pass / (peaks["hbm_gbs"] * 1e9) * 1e3
    t_cmp = flops_per_pass / (peak_tf * 1e12) * 1e3
    if t_hbm > t_cmp:
        bound, unit = "hbm", "GB/s"
        achieved = bytes_per_pass / (avg_pass / 1e3) / 1e9
        peak = peaks["hbm_gbs"]
        basis = f"{peaks_src} HBM copy bandwidth"
    else:
        peak = peak_tf
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic_latest.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"{args.config}:{contract}")
        except Exception:
            traffic = None
    if args.variant in ("uniform", "leverage"):
        # rSTR-U / -L: no dense pass; the HBM traffic of a step is the zipped-fiber gathers X_S[n]
        # (m fibers per mode).  Sector bytes: mode 1 fibers are contiguous (ceil(I_1 b / 32) sectors),
        # every other mode's fiber elements sit in separate 32-byte sectors.  Bound = those bytes /
        # HBM bandwidth, against the whole step (the step is latency-bound: small GEMMs and solves).
        m = cfg.sketch_rows or 2000
        xb = 4 if cfg.dtype == "f32" else 8
        dims_t = list(cfg.dims) + [cfg.t_new]
        dims_t[0] = dims_t[0] // world
        sectors = -(-dims_t[0] * xb // 32) + sum(dims_t[1:])
        sec_bytes = m * 32 * sectors
        useful = m * xb * sum(dims_t)
        step_s = ms / args.steps / 1e3
        ach = sec_bytes / step_s / 1e9
        roofline = {"bound": "hbm", "achieved": round(ach, 3), "peak": round(peaks["hbm_gbs"], 3), "unit": "GB/s",
                    "frac": round(ach / peaks["hbm_gbs"], 5), "traffic": None,
                    "kernel": "whole rSTR step over its gathered fiber sectors (no dense pass on the path)",
                    "algorithmic_per_step": {"sector_bytes": sec_bytes, "useful_bytes": useful},
                    "t_hbm_floor_us": round(sec_bytes / (peaks["hbm_gbs"] * 1e9) * 1e6, 3),
                    "peak_basis": f"{peaks_src} HBM copy bandwidth"}
    elif args.variant == "ksrft":
        # rSTR-K: the dominant kernels are the N KSRFT mixing passes over the batch (HBM-bound):
        # algorithmic bytes = |X| (in + 8 B complex out) for mode 1 + 16 B per entry for modes 2..N
        mix_ms = p1_ms / max(p1_n, 1)
        xb = 4 if cfg.dtype == "f32" else 8
        cb = 8 if contract == "3xtf32" else 16
        mix_bytes = local_entries * ((xb + cb) + 2 * cb * (cfg.N - 1))
        ksrft_traffic = None   # DRAM bytes of the N passes from one ncu --set full capture (tools/save_profiles.py)
        if os.path.exists(tpath):
            try:
                ksrft_traffic = json.load(open(tpath)).get(f"{cfg.name}:ksrft")
            except Exception:
                ksrft_traffic = None
        ach = mix_bytes / (mix_ms / 1e3) / 1e9
        roofline = {"bound": "hbm", "achieved": round(ach, 3), "peak": round(peaks["hbm_gbs"], 3), "unit": "GB/s",
                    "frac": round(ach / peaks["hbm_gbs"], 4), "traffic": ksrft_traffic,
                    "kernel": f"KSRFT mixing ({cfg.N} passes, events around the span)",
                    "mix_us": round(mix_ms * 1e3, 2),
                    "mix_share_of_step": round(mix_ms / (ms / args.steps), 4),
                    "algorithmic_per_launch": {"bytes": mix_bytes}, "peak_basis": f"{peaks_src} HBM copy bandwidth"}
    else:
      roofline = {"bound": bound, "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": unit,
                  "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": "contraction pass (avg of pass 1/2)",
                  "pass1_us": round(avg_p1 * 1e3, 2), "pass2_us": round(avg_p2 * 1e3, 2),
                  "pass_share_of_step": round((p1_ms + p2_ms) / max(kp, 1) / (ms / args.steps), 4),
                  "algorithmic_per_launch": {"flops": flops_per_pass, "bytes": bytes_per_pass},
                  "peak_basis": basis,
                  "frac_vs_other_peaks": ({k: round(achieved / v, 4) for k, v in alt.items()}
                                          if unit == "TFLOP/s" else {}),
                  # step-level fraction: the two passes' algorithmic minimum (F_min, or their bytes when
                  # HBM-bound) over the whole step at this peak
                  "step_frac": round((2 * flops_per_pass / 1e12 if unit == "TFLOP/s" else 2 * bytes_per_pass / 1e9)
                                     / (ms / args.steps / 1e3) / peak, 4),
                  # the paper's mode-by-mode work F_paper = N 2|X|R^2 per step vs the
                  # two-pass F_min = 2 passes x 2|X|R^2, both over the measured step time
                  "per_step": {"F_min": 2 * flops_per_pass, "F_paper": cfg.N * flops_per_pass,
                               "F_min_tflops_over_step": round(2 * flops_per_pass / (ms / args.steps / 1e3) / 1e12, 3),
                               "F_paper_tflops_over_step": round(cfg.N * flops_per_pass / (ms / args.steps / 1e3) / 1e12, 3)}}
    if args.variant == "det" and span and all(x for x in span):
        # in-kernel span (first CTA start to last CTA end, %globaltimer) of the last profiled step;
        # the event pair above also holds the graph node's launch latency (~6 us measured with an
        # empty kernel in the same position)
        sp = 0.5 * (span[0] + span[1])
        ach_sp = (flops_per_pass if unit == "TFLOP/s" else bytes_per_pass) / (sp / 1e6) / (1e12 if unit == "TFLOP/s" else 1e9)
        roofline["kernel_span_us"] = {"pass1": round(span[0], 2), "pass2": round(span[1], 2)}
        roofline["achieved_kernel_span"] = round(ach_sp, 3)
        roofline["frac_kernel_span"] = round(ach_sp / peak, 4)

    # ---- e2e: public host-buffer API, pinned H2D + D2H of the step's result every step
    pinned = [torch.from_numpy(x).pin_memory() for x in host[:min(nd, 4)]]
    res = np.empty((cfg.t_new, R2))
    for i in range(2):
        lib.str_update_batch_host(h, pinned[i % len(pinned)], cfg.t_new)
        res = lib.str_get_temporal_rows(h, lib.str_processed(h) - cfg.t_new, cfg.t_new)
    barrier()
    torch.cuda.synchronize(dev)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for i in range(args.e2e_steps):
        lib.str_update_batch_host(h, pinned[i % len(pinned)], cfg.t_new)
        res = lib.str_get_temporal_rows(h, lib.str_processed(h) - cfg.t_new, cfg.t_new)
    f1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    e2e_ms = maxall(f0.elapsed_time(f1))
    e2e = {"value": args.e2e_steps * global_entries / (e2e_ms / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": int(pinned[0].numel() * pinned[0].element_size()),
           "d2h_bytes_per_step": int(res.size * 8), "steps": args.e2e_steps}
    # the step's batch crosses the host link inside the timed region and the result read waits for the
    # step, so copy and compute are serialized: e2e is bound by the H2D copy, not by the library
    e2e["h2d_gb_per_s"] = round(e2e["h2d_bytes_per_step"] * args.e2e_steps / (e2e_ms / 1e3) / 1e9, 2)
    e2e["ms_per_step"] = round(e2e_ms / args.e2e_steps, 4)
    e2e["bound"] = "host link: pinned H2D of the batch each step, serialized with the step by the result read"
    # ---- batch TR-ALS on the init slab (Alg. 1, the initialization stage; not part of the step)
    tr_als = None
    if world == 1 and args.variant == "det":
        Xi_d = torch.from_numpy(Xi).to(dev)
        torch.cuda.synchronize(dev)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sw = 2
        lib.str_tr_als(h, Xi_d, cfg.t_init, 1)   # warm-up (captures the sweep graph)
        a0.record(stream)
        fit = lib.str_tr_als(h, Xi_d, cfg.t_init, sw)
        a1.record(stream)
        torch.cuda.synchronize(dev)
        tr_als = {"sweeps": sw, "t": cfg.t_init, "ms_per_sweep": round(a0.elapsed_time(a1) / sw, 4),
                  "note": "includes the rebuild of the streaming state and one fit evaluation", "fit": fit}
    lib.str_destroy(h)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "3xtf32+f64" if contract == "3xtf32" else "f64",
            "data": "synthetic (seeded TR stream, SURVEY.md §8(d).1)",
            "config": {"workload": f"{cfg.name}: order-{cfg.N} {'x'.join(map(str, cfg.dims))} x t_new={cfg.t_new} "
                                   f"{cfg.dtype}, TR ranks {cfg.ranks[0]}, "
                                   + ("STR (Alg. 4)" if args.variant == "det" else
                                      f"rSTR-{ {'uniform': 'U', 'leverage': 'L', 'ksrft': 'K'}[args.variant]} "
                                      f"(Alg. { {'uniform': 7, 'leverage': 8, 'ksrft': 9}[args.variant]}), "
                                      f"m = {cfg.sketch_rows or 2000}") + ", X_new sharded on mode 1",
                       "global_batch_entries": global_entries, "contract": contract, "split_k": cfg.split_k,
                       "parallelism": f"mode-1 shard x{world}",
                       "l2": f"rotating {nd} distinct device-resident batches ({nd * global_entries * 4 / 1e9:.2f} GB)"
                             " > 126 MB L2"},
            "gpu_launches": int(launches), "clocks": clk.summary(), "e2e": e2e, "roofline": roofline,
            "latency": latency}
    if tr_als:
        line["tr_als_init"] = tr_als
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, variant=args.variant)
    if world > 1:
        line["nccl"] = nccl_summary(nccl_glob) if nccl_glob else None
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def oracle_stream(cfg, variant, s):
    """The oracle of the benched variant: STR (Alg. 4), rSTR-U / -L (Alg. 7 / 8), rSTR-K (Alg. 9)."""
    from workloads.gen import paper_view
    Xi = paper_view(s.init_slab())
    m = cfg.sketch_rows or 2000
    if variant == "det":
        from oracle.stream import StreamingTR
        return StreamingTR(Xi, s.init_cores())
    if variant == "ksrft":
        from oracle.ksrft import KSRFTStreamingTR
        return KSRFTStreamingTR(Xi, s.init_cores(), m, cfg.seed)
    from oracle.rstream import RandomizedStreamingTR
    return RandomizedStreamingTR(Xi, s.init_cores(), m, variant, cfg.seed)


def cpu_baseline(cfg, budget_s=20.0, variant="det"):
    """The oracle as it stands (fp64 numpy) on this host's cores: init + update steps on the
    same workload until ~budget_s of update time; value = entries / update seconds."""
    from workloads import make_stream
    from workloads.gen import paper_view
    s = make_stream(cfg)
    st = oracle_stream(cfg, variant, s)
    t_used, steps = 0.0, 0
    while t_used < budget_s and steps < cfg.n_batches:
        Xb = paper_view(s.batch(steps))
        t = time.perf_counter()
        st.update(Xb)
        t_used += time.perf_counter() - t
        steps += 1
    hi = host_info()
    return {"value": steps * cfg.batch_entries / t_used, "unit": UNIT, "cores": hi["blas_threads"], "kind": "oracle",
            "sample": f"{cfg.name} ({variant}): oracle init + {steps} full update steps ({t_used:.1f} s of update time; "
                      f"numpy BLAS threads = {hi['blas_threads']} of {hi['host_cores']} host cores)",
            "host": hi}


def bench_reference(args):
    """--impl reference: the oracle (fp64 CPU, as it stands) on the same workload/metric."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from workloads import get_config, make_stream
    from workloads.gen import paper_view
    cfg = get_config(args.config)
    s = make_stream(cfg)
    st = oracle_stream(cfg, args.variant, s)
    nd = min(N_DISTINCT, cfg.n_batches)
    for w in range(min(args.warmup, 1)):
        st.update(paper_view(s.batch(w % nd)))
    t_used, steps = 0.0, 0
    while steps < args.steps and (t_used < args.ref_budget or steps == 0):
        Xb = paper_view(s.batch(steps % nd))
        t = time.perf_counter()
        st.update(Xb)
        t_used += time.perf_counter() - t
        steps += 1
    value = steps * cfg.batch_entries / t_used
    sample = (f"{cfg.name}: {steps} of the requested {args.steps} oracle update steps "
              f"(time budget {args.ref_budget:.0f} s), warm-up {min(args.warmup, 1)}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": steps, "warmup": min(args.warmup, 1), "ms_per_step": 1e3 * t_used / steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded TR stream, SURVEY.md §8(d).1)",
            "config": {"workload": f"{cfg.name} (same as ours), variant {args.variant}",
                       "global_batch_entries": cfg.batch_entries},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": host_info()["blas_threads"], "kind": "oracle",
                             "sample": sample, "host": host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--contract", default=None, choices=[None, "3xtf32", "f64"])
    ap.add_argument("--variant", default="det", choices=["det", "uniform", "leverage", "ksrft"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--ref-budget", type=float, default=60.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--split-k", type=int, default=None, help="two-pass split point k (default: the config's)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
