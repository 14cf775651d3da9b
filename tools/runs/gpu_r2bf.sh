#!/bin/bash
# factor on a two-CTA cluster (V rows on the second CTA, pushed L/T) vs one CTA (STR_FACTOR_SPLIT=0)
python paper_2307_00719_b200/build.py 2>&1 | tail -1
(cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DFC_PROBE -I../../include -I../../paper_2307_00719_b200/csrc -o fc_probe fc_probe.cu && timeout 60 ./fc_probe 100 && timeout 60 ./fc_probe 64 && STR_FACTOR_SPLIT=0 timeout 60 ./fc_probe 100) > gpurun_out/r2bf_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spd_inv.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2bf_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2bf_pytest.log
for c in C5 C4 C3; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2bf_b_$c.log 2>&1; done
STR_FACTOR_SPLIT=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C5 > gpurun_out/r2bf_b0_C5.log 2>&1
