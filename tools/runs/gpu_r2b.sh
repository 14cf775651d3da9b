#!/bin/bash
# new SPD inverse: unit test, parity subset, step time A/B (STR_INV=0 old cluster sweep)
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_spd_inv.py tests/test_gpu_parity.py tests/test_gpu_rstr.py tests/test_gpu_traj.py -x -q -s -p no:cacheprovider -k "not pert" > gpurun_out/r2b_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
for inv in 0 1; do
  STR_INV=$inv timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2b_bench_inv$inv.log 2>&1
  echo "rc=$?" >> gpurun_out/r2b_bench_inv$inv.log
done
STR_INV=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config C4 > gpurun_out/r2b_bench_c4.log 2>&1
