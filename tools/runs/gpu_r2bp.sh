#!/bin/bash
# two-CTA factor also at S = 64 (C4 STR / rSTR)
python paper_2307_00719_b200/build.py 2>&1 | tail -1
(cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DFC_PROBE -I../../include -I../../paper_2307_00719_b200/csrc -o fc_probe fc_probe.cu && timeout 60 ./fc_probe 64 && STR_FACTOR_SPLIT=0 timeout 60 ./fc_probe 64) > gpurun_out/r2bp_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spd_inv.py tests/test_gpu_parity.py tests/test_gpu_rstr.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2bp_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2bp_pytest.log
for v in det uniform leverage; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant $v > gpurun_out/r2bp_C4_$v.log 2>&1; done
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C2 > gpurun_out/r2bp_C2.log 2>&1
