#!/bin/bash
# factor: pivot warp alone on its SM sub-partition (FC_EXCL) x thread counts; tests; bench
python paper_2307_00719_b200/build.py 2>&1 | tail -1
(cd tools/micro && for v in "384 1" "512 1" "384 0" "256 1"; do set -- $v; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DFC_PROBE -DFC_THREADS=$1 -DFC_EXCL=$2 -I../../include -I../../paper_2307_00719_b200/csrc -o fc_probe_$1_$2 fc_probe.cu && echo "== threads $1 excl $2" && ./fc_probe_$1_$2 100 && ./fc_probe_$1_$2 64; done) > gpurun_out/r2x_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spd_inv.py tests/test_gpu_parity.py tests/test_gpu_loopback.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2x_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2x_pytest.log
for c in C5 C4; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2x_b_$c.log 2>&1; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant uniform > gpurun_out/r2x_b_C4u.log 2>&1
