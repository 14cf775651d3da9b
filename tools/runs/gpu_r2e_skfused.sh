#!/bin/bash
# split-K GEMM with the reduce fused (last CTA per tile): rSTR parity subset + A/B bench lines, then the final evidence pass
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_rstr.py tests/test_gpu_ksrft.py -m gpu -q -x -p no:cacheprovider > gpurun_out/skf_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/skf_pytest.log
for v in uniform leverage ksrft; do
  STR_SK_FUSED=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant $v > gpurun_out/skf_off_$v.log 2>&1
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant $v > gpurun_out/skf_on_$v.log 2>&1
done
bash tools/runs/gpu_r2e_final.sh
