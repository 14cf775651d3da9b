#!/bin/bash
# factor: batched symmetrise + 11 worker warps; probe (384 vs 256 vs 512 threads), tests, bench
python paper_2307_00719_b200/build.py 2>&1 | tail -1
(cd tools/micro && for T in 256 384 512; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DFC_PROBE -DFC_THREADS=$T -I../../include -I../../paper_2307_00719_b200/csrc -o fc_probe_$T fc_probe.cu && echo "== threads $T" && ./fc_probe_$T 100 && ./fc_probe_$T 64; done) > gpurun_out/r2u_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spd_inv.py tests/test_gpu_parity.py tests/test_gpu_loopback.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2u_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2u_pytest.log
for c in C5 C4; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2u_b_$c.log 2>&1; done
