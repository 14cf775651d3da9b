#!/bin/bash
# FP64 contraction: wave-aware split-K count (whole waves of 2 x 148 CTAs): FP64 parity + bench lines
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C5 --contract f64 > gpurun_out/fw_c5.log 2>&1
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C3 > gpurun_out/fw_c3.log 2>&1
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --contract f64 > gpurun_out/fw_c4.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_traj.py tests/test_gpu_sweeps.py tests/test_gpu_contract.py -m gpu -q -p no:cacheprovider -k "f64 or F64 or fp64 or C3 or c3" > gpurun_out/fw_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/fw_pytest.log
