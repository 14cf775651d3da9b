#!/bin/bash
# chain GEMM: absorb accumulate: old P values loaded at kernel start
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_trals.py tests/test_gpu_loopback.py tests/test_gpu_traj.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2av_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2av_pytest.log
for c in C5 C4 C2; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2av_b_$c.log 2>&1; done
timeout 300 python tools/graphtrace.py C5 --prof > gpurun_out/r2av_gt_C5.log 2>&1
timeout 300 python tools/graphtrace.py C4 --prof > gpurun_out/r2av_gt_C4.log 2>&1
