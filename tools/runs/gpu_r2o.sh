#!/bin/bash
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_trals.py tests/test_gpu_contract.py tests/test_gpu_loopback.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/r2o_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2o_pytest.log
for c in C5 C4 C3 C2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2o_bench_$c.log 2>&1; done
