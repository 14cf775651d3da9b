#!/bin/bash
# dynamic unit schedule of the contraction: correctness, then static-share / chunk sweep
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_contract.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2t_pytest.log 2>&1
rc=$?
echo "rc=$rc" >> gpurun_out/r2t_pytest.log
[ $rc -ne 0 ] && exit 1
for cfg in "100 2" "80 2" "70 2" "80 1" "80 4" "90 2"; do
  set -- $cfg
  for c in C5 C4; do
    STR_TF_STATIC=$1 STR_TF_DCHUNK=$2 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2t_b_${c}_$1_$2.log 2>&1
  done
done
