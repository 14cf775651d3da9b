#!/bin/bash
# FP64 contraction split-K target CTA count sweep (C3, C5 FP64)
python paper_2307_00719_b200/build.py 2>&1 | tail -1
for n in 296 148 74 592; do
  STR_F64_CTAS=$n timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C3 > gpurun_out/r2bl_C3_$n.log 2>&1
  STR_F64_CTAS=$n timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C5 --contract f64 > gpurun_out/r2bl_C5f_$n.log 2>&1
done
