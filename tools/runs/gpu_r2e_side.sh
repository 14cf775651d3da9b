#!/bin/bash
# ncu --set full of the step's secondary kernels (absorbs, chain GEMMs, factor, rows, tables) at C5 and the
# rSTR-U launch list at C4 (evidence for the latency-bound classes of DESIGN §4 / §11)
python paper_2307_00719_b200/build.py 2>&1 | tail -1
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2"
timeout 300 $CMD > gpurun_out/side_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_absorb6|k_chain_gemm|k_spd_factor|k_rows_solve|k_build_table3" -s 117 -c 39 -o gpurun_out/prof_side $CMD > gpurun_out/side_ncu.log 2>&1
CMDU="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 --config C4 --variant uniform"
timeout 300 $CMDU > gpurun_out/side_plain_u.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rstr_u.csv $CMDU > gpurun_out/side_ncu_u.log 2>&1
