#!/bin/bash
# serial chain on its own stream (programmatic edges), data stream hands over P_j / B_{j+1}
python paper_2307_00719_b200/build.py 2>&1 | tail -1
for c in C5 C4 C2 C3; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2aa_b_$c.log 2>&1; done
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2aa_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2aa_pytest.log
timeout 300 python tools/loopback_stress.py > gpurun_out/r2aa_stress.log 2>&1; echo "rc=$?" >> gpurun_out/r2aa_stress.log
