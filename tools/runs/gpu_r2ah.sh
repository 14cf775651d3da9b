#!/bin/bash
# rows+Gram cluster kernel with overlapped DSMEM reduction: A/B vs two kernels; table ring depth 3 re-check; C4 pass trace
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2ah_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2ah_pytest.log
for c in C5 C4; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2ah_b_$c.log 2>&1; done
for c in C5 C4; do STR_FUSE_RG=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2ah_b0_$c.log 2>&1; done
for c in C5 C4; do STR_FUSE_RG=0 STR_TF_BSTAGES=3 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/r2ah_b3_$c.log 2>&1; done
STR_FUSE_RG=0 timeout 300 python tools/timeline.py --config C5 > gpurun_out/r2ah_tl_C5_0.log 2>&1
timeout 300 python tools/timeline.py --config C5 > gpurun_out/r2ah_tl_C5_1.log 2>&1
STR_FUSE_RG=0 timeout 300 python tools/graphtrace.py C4 --prof > gpurun_out/r2ah_gt_C4.log 2>&1
