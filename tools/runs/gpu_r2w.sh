#!/bin/bash
# factor: symmetrised lower triangle loaded straight from global; probe, tests, bench
python paper_2307_00719_b200/build.py 2>&1 | tail -1
(cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DFC_PROBE -I../../include -I../../paper_2307_00719_b200/csrc -o fc_probe fc_probe.cu && ./fc_probe 100 && ./fc_probe 64) > gpurun_out/r2w_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spd_inv.py tests/test_gpu_parity.py tests/test_gpu_loopback.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2w_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2w_pytest.log
for c in C5 C4; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2w_b_$c.log 2>&1; done
