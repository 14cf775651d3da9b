#!/bin/bash
# rSTR: fiber gather on the side stream beside the sampled chain: parity subset + bench lines (compare with skf_on_* of gpu_r2f.sh), then the final evidence pass
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_rstr.py tests/test_gpu_ksrft.py tests/test_gpu_stress.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gs_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gs_pytest.log
for v in uniform leverage ksrft; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant $v > gpurun_out/gs_$v.log 2>&1
done
bash tools/runs/gpu_r2e_final.sh
