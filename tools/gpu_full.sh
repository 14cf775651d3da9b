#!/bin/bash
# full GPU suite + smoke + bench (C5 default line) + C4/C3/C2 and rSTR bench lines
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/full_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/full_pytest.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/full_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/full_smoke.log
timeout 600 python bench.py > gpurun_out/full_bench_c5.log 2>&1
for c in C4 C3 C2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/full_bench_$c.log 2>&1; done
for v in uniform leverage ksrft; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant $v > gpurun_out/full_bench_c4_$v.log 2>&1; done
