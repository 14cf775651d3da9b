python paper_2307_00719_b200/build.py 2>&1 | tail -1
STR_INV=0 timeout 300 python -m pytest tests/test_gpu_spd_inv.py -q -x 2>&1 | grep -E "Error|assert|passed|failed" | head -8 > gpurun_out/r2i.log

