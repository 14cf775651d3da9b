#!/bin/bash
python paper_2307_00719_b200/build.py 2>&1 | tail -1
python tools/ncu_small.py uniform > gpurun_out/r2r_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_sampled_accum|k_spd_factor|k_reduce_sk" -s 8 -c 3 -o gpurun_out/r2r_small python tools/ncu_small.py uniform > gpurun_out/r2r_ncu.log 2>&1
