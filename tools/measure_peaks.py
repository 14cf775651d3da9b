#!/usr/bin/env python
"""Measured TF32 and FP64 matmul peaks on this GPU (the roofline denominators bench.py needs for the
3xTF32 and FP64 contraction kernels; MEASURED_PEAKS.json only has HBM and bf16).

cuBLAS via torch.matmul, 8192^3 (2 N^3 flops): best of 10 launches (burst) and back to back for
~3 s (sustained), CUDA events.  TF32 = fp32 operands with allow_tf32 (tcgen05 kind::tf32).
Writes one JSON object to the path given (default gpurun_out/measured_peaks.json).
"""
import json
import sys
import time

import torch


def gemm_peak(dtype, tf32, n=8192, sustain_s=3.0):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    c = torch.empty(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    # sustained: back to back for ~sustain_s
    reps = max(10, int(sustain_s * 1e3 / best))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        torch.matmul(a, b, out=c)
    e1.record()
    torch.cuda.synchronize()
    sus = e0.elapsed_time(e1) / reps
    f = 2.0 * n ** 3
    return {"burst_tflops": round(f / (best / 1e3) / 1e12, 1), "sustained_tflops": round(f / (sus / 1e3) / 1e12, 1),
            "n": n, "reps_sustained": reps}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/measured_peaks.json"
    res = {"gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "how": "cuBLAS via torch.matmul 8192^3 (2 N^3 flops): best of 10 (burst), back to back ~3 s (sustained)",
           "tf32": gemm_peak(torch.float32, True),
           "fp32_ffma": gemm_peak(torch.float32, False, n=4096, sustain_s=1.5),
           "fp64": gemm_peak(torch.float64, False, n=4096, sustain_s=2.0)}
    print(json.dumps(res))
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
