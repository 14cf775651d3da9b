#!/bin/bash
python paper_2307_00719_b200/build.py 2>&1 | tail -1
for inv in 0 1; do echo "STR_INV=$inv"; STR_INV=$inv python tools/inv_time.py; STR_INV=$inv timeout 300 python -m pytest tests/test_gpu_spd_inv.py -q -x 2>&1 | tail -1; done > gpurun_out/r2h_inv.log 2>&1
for inv in 0 1; do
  STR_INV=$inv timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r2h_bench_inv$inv.log 2>&1
done
STR_INV=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 > gpurun_out/r2h_bench_c4.log 2>&1
