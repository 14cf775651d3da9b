#!/bin/bash
# what-if on the diagnostic build at the r2ad factor (skip masks: 1 factor, 2 tables, 4 passes, 8 absorbs, 16 chain GEMMs, 32 rows, 64 Grams)
bash tools/gpu_whatif2.sh > gpurun_out/r2af_whatif.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spd_inv.py tests/test_gpu_parity.py tests/test_gpu_traj.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2af_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2af_pytest.log
