#!/bin/bash
# two-pass split point k at C5 / C4 (bench --split-k)
python paper_2307_00719_b200/build.py 2>&1 | tail -1
for k in 1 2 3; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C5 --split-k $k > gpurun_out/r2bo_C5_k$k.log 2>&1; done
for k in 1 2; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --split-k $k > gpurun_out/r2bo_C4_k$k.log 2>&1; done
