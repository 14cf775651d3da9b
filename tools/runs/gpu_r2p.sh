#!/bin/bash
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_rstr.py tests/test_gpu_ksrft.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r2p_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2p_pytest.log
for c in C5 C4; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2p_bench_$c.log 2>&1; done
for v in uniform leverage; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant $v > gpurun_out/r2p_bench_c4_$v.log 2>&1; done
