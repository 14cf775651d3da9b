#!/bin/bash
# merged MMA commit (A slot + table slot) A/B, fused pass-2 generation profile
python paper_2307_00719_b200/build.py 2>&1 | tail -1
B="python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2"
STR_TF_GEN=0 timeout 300 $B > gpurun_out/c2_c5_merge.log 2>&1
STR_TF_GEN=0 STR_TF_MERGE=0 timeout 300 $B > gpurun_out/c2_c5_nomerge.log 2>&1
timeout 300 $B > gpurun_out/c2_c5_gen_merge.log 2>&1
timeout 300 $B --config C4 > gpurun_out/c2_c4_merge.log 2>&1
STR_TF_MERGE=0 timeout 300 $B --config C4 > gpurun_out/c2_c4_nomerge.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fused_table.py tests/test_gpu_contract.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/c2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/c2_pytest.log
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:ILi2ELi10E -s 3 -c 1 -o gpurun_out/c2_gen python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c2_ncu.log 2>&1
