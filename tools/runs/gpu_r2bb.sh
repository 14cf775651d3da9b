#!/bin/bash
# factor: V = L^{-1} by recursive doubling after the factorization (FC_VREC) vs V rows in the step loop
python paper_2307_00719_b200/build.py 2>&1 | tail -1
(cd tools/micro && for v in 0 1; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DFC_PROBE -DFC_VREC=$v -I../../include -I../../paper_2307_00719_b200/csrc -o fcv_$v fc_probe.cu && echo "== vrec $v" && ./fcv_$v 100 && ./fcv_$v 64; done) > gpurun_out/r2bb_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spd_inv.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2bb_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2bb_pytest.log
for c in C5 C4; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2bb_b_$c.log 2>&1; done
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant uniform > gpurun_out/r2bb_b_C4u.log 2>&1
