#!/bin/bash
python paper_2307_00719_b200/build.py 2>&1 | tail -1
(cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DFC_PROBE -I../../include -I../../paper_2307_00719_b200/csrc -o fc_probe fc_probe.cu && for S in 25 64 100 128; do ./fc_probe $S; done) > gpurun_out/r2j_probe.log 2>&1
python tools/inv_time.py >> gpurun_out/r2j_probe.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_spd_inv.py tests/test_gpu_parity.py tests/test_gpu_traj.py tests/test_gpu_rstr.py tests/test_gpu_trals.py tests/test_gpu_edges.py tests/test_gpu_loopback.py -x -q -s -p no:cacheprovider > gpurun_out/r2j_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2j_pytest.log
for c in C5 C4 C3 C2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2j_bench_$c.log 2>&1; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant uniform > gpurun_out/r2j_bench_c4u.log 2>&1
