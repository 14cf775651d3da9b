#!/bin/bash
# re-entry baseline at HEAD: full GPU suite, smoke, C5 + C4 bench lines
python paper_2307_00719_b200/build.py 2>&1 | tail -1
nvidia-smi -L
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c0_bench_c5.log 2>&1
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 > gpurun_out/c0_bench_c4.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/c0_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/c0_pytest.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c0_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/c0_smoke.log
