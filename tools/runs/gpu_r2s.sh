#!/bin/bash
# fork ordering A/B (pass-1 created before the side branch) + measured TF32/FP64 peaks
python paper_2307_00719_b200/build.py 2>&1 | tail -1
python tools/measure_peaks.py gpurun_out/measured_peaks.json > gpurun_out/r2s_peaks.log 2>&1
timeout 600 python -m pytest tests/test_gpu_traj.py tests/test_gpu_loopback.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2s_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2s_pytest.log
for i in 1 2; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r2s_bench_c5_$i.log 2>&1; done
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 > gpurun_out/r2s_bench_c4.log 2>&1
