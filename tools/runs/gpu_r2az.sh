#!/bin/bash
# rSTR: split-K reduce loads the accumulated value before the PDL wait
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_rstr.py tests/test_gpu_ksrft.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2az_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2az_pytest.log
for v in uniform leverage ksrft; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant $v > gpurun_out/r2az_b_$v.log 2>&1; done
