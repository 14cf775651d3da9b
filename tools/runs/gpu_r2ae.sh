#!/bin/bash
# factor: pivot warp loads its block before releasing the workers (FC_WAITFIRST 1 / 0 probe), tests, benches
python paper_2307_00719_b200/build.py 2>&1 | tail -1
(cd tools/micro && for w in 1 0; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DFC_PROBE -DFC_WAITFIRST=$w -I../../include -I../../paper_2307_00719_b200/csrc -o fc_probe_$w fc_probe.cu && echo "== waitfirst $w" && ./fc_probe_$w 100 && ./fc_probe_$w 64; done) > gpurun_out/r2ae_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spd_inv.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2ae_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2ae_pytest.log
for c in C5 C4; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2ae_b_$c.log 2>&1; done
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant uniform > gpurun_out/r2ae_b_C4u.log 2>&1
