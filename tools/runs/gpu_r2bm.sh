#!/bin/bash
# FP64 contraction: K chunks capped at ~640 (more splits for large-K passes)
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_contract.py tests/test_gpu_traj.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2bm_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2bm_pytest.log
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C3 > gpurun_out/r2bm_b_C3.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C5 --contract f64 > gpurun_out/r2bm_b_C5f.log 2>&1
