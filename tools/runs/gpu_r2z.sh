#!/bin/bash
# gate A/B and pass-1 grid with the gate
python paper_2307_00719_b200/build.py 2>&1 | tail -1
for v in "0 0" "1 0" "1 136" "1 128" "1 120" "0 0"; do
  set -- $v
  for c in C5 C4; do
    if [ $2 -eq 0 ]; then STR_GATE=$1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2z_b_${c}_$1_$2.log 2>&1
    else STR_GATE=$1 STR_TF_GRID=$2 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2z_b_${c}_$1_$2.log 2>&1; fi
  done
done
