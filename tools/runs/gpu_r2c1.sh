#!/bin/bash
# fused pass-2 table generation: parity first (C5 + contract hooks), then bench with/without, and the UMMA rate probe
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_fused_table.py tests/test_gpu_contract.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/c1_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/c1_pytest.log
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c1_bench_gen.log 2>&1
STR_TF_GEN=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c1_bench_nogen.log 2>&1
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c1_bench_gen2.log 2>&1
(cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_probe umma_probe.cu && timeout 60 ./umma_probe) > gpurun_out/c1_umma.log 2>&1
