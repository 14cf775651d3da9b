#!/bin/bash
# rows + Gram fused in one cluster launch (k_rows_gram): parity, benches A/B (STR_FUSE_RG=0)
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_loopback.py tests/test_gpu_trals.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2ag_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2ag_pytest.log
for c in C5 C4 C3 C2; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2ag_b_$c.log 2>&1; done
for c in C5 C4; do STR_FUSE_RG=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2ag_b0_$c.log 2>&1; done
timeout 1200 python -m pytest tests/test_gpu_traj.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2ag_pytest2.log 2>&1
echo "rc=$?" >> gpurun_out/r2ag_pytest2.log
