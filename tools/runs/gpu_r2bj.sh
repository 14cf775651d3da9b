#!/bin/bash
# M_N by one absorb over the left multi-index with the left-group table (k >= 2)
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_trals.py tests/test_gpu_loopback.py tests/test_gpu_traj.py tests/test_gpu_sweeps.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2bj_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2bj_pytest.log
for c in C5 C4 C2 C3; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2bj_b_$c.log 2>&1; done
