#!/bin/bash
# contraction epilogue: wait only for the staging reads at exit; staging rows padded to 4 (mod 32) floats
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_contract.py tests/test_gpu_parity.py tests/test_gpu_sweeps.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2as_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2as_pytest.log
for c in C5 C4 C2; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2as_b_$c.log 2>&1; done
timeout 300 python tools/graphtrace.py C5 --prof > gpurun_out/r2as_gt_C5.log 2>&1
timeout 300 python tools/graphtrace.py C4 --prof > gpurun_out/r2as_gt_C4.log 2>&1
