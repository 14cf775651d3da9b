#!/bin/bash
# event-pair overhead by kernel shape (launch_probe) + C5 pass trace
python paper_2307_00719_b200/build.py 2>&1 | tail -1
(cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_probe launch_probe.cu && ./launch_probe) > gpurun_out/r2ai_launch.log 2>&1
timeout 300 python tools/graphtrace.py C5 --prof > gpurun_out/r2ai_gt_C5.log 2>&1
