#!/bin/bash
# round-2 validation: full GPU suite (minus the cached-C5 trajectories) + bench
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q -k "not C5_every_batch" -s -p no:cacheprovider > gpurun_out/r2a_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2a_bench.log
