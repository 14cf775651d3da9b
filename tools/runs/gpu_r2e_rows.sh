#!/bin/bash
# rows solve on 16 warps / two accumulator chains: solve + parity subset, C5/C4/C3/rSTR-U bench lines; then the side-kernel profile
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_spd_inv.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_rstr.py -m gpu -q -x -p no:cacheprovider > gpurun_out/rows_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/rows_pytest.log
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/rows_c5.log 2>&1
for c in C4 C3; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/rows_${c,,}.log 2>&1; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant uniform > gpurun_out/rows_rstr_u.log 2>&1
bash tools/runs/gpu_r2e_side.sh
