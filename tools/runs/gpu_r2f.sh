#!/bin/bash
python paper_2307_00719_b200/build.py 2>&1 | tail -1
(cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DFC_PROBE -I../../include -I../../paper_2307_00719_b200/csrc -o fc_probe fc_probe.cu && for S in 25 64 100 128; do ./fc_probe $S; done) > gpurun_out/r2f_probe.log 2>&1
timeout 300 python -m pytest tests/test_gpu_spd_inv.py -q -x > gpurun_out/r2f_pytest.log 2>&1
python tools/inv_time.py >> gpurun_out/r2f_pytest.log 2>&1
timeout 600 python tools/loopback_stress.py > gpurun_out/r2f_stress.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r2f_bench.log 2>&1
