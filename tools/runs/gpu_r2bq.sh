#!/bin/bash
# rSTR-U: draws + sampled-row gather fused into the rows solve
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_rstr.py tests/test_gpu_ksrft.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2bq_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2bq_pytest.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2bq_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2bq_smoke.log
for v in uniform leverage; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant $v > gpurun_out/r2bq_C4_$v.log 2>&1; done
