#!/bin/bash
# fused pass-2 generation v3 (next unit's G_k slice prefetched, one division per row): parity + A/B
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_fused_table.py tests/test_gpu_contract.py -x -q -p no:cacheprovider > gpurun_out/c4_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/c4_pytest.log
B="python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2"
STR_TF_GEN=1 timeout 300 $B > gpurun_out/c4_gen.log 2>&1
timeout 300 $B > gpurun_out/c4_default.log 2>&1
