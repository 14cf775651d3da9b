#!/bin/bash
# fused pass-2 generation v2 (4 generator warps, cp.async prefix staging): parity + A/B bench
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_fused_table.py tests/test_gpu_contract.py -x -q -p no:cacheprovider > gpurun_out/c3_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/c3_pytest.log
B="python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2"
timeout 300 $B > gpurun_out/c3_gen.log 2>&1
STR_TF_GEN=0 timeout 300 $B > gpurun_out/c3_nogen.log 2>&1
timeout 300 $B > gpurun_out/c3_gen2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:ILi2ELi10E -s 3 -c 1 -o gpurun_out/c3_gen python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c3_ncu.log 2>&1
