#!/bin/bash
python paper_2307_00719_b200/build.py 2>&1 | tail -1
(cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DFC_PROBE -I../../include -I../../paper_2307_00719_b200/csrc -o fc_probe fc_probe.cu && for S in 25 64 100 128; do ./fc_probe $S; done) > gpurun_out/r2d_probe.log 2>&1
timeout 600 python -m pytest tests/test_gpu_loopback.py -x -q -s -p no:cacheprovider > gpurun_out/r2d_loopback.log 2>&1
echo "rc=$?" >> gpurun_out/r2d_loopback.log
