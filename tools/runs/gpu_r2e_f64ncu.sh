#!/bin/bash
# ncu --set full of the FP64 (DMMA) contraction at C5 (--contract f64) and C3 (its production path)
python paper_2307_00719_b200/build.py 2>&1 | tail -1
CMD5="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 --config C5 --contract f64"
CMD3="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 --config C3"
timeout 300 $CMD5 > gpurun_out/f64_plain5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_contract_f64 -s 6 -c 2 -o gpurun_out/prof_f64_c5 $CMD5 > gpurun_out/f64_ncu5.log 2>&1
timeout 300 $CMD3 > gpurun_out/f64_plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_contract_f64 -s 6 -c 2 -o gpurun_out/prof_f64_c3 $CMD3 > gpurun_out/f64_ncu3.log 2>&1
