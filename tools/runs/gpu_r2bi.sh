#!/bin/bash
# kernel-boundary cost: chains of empty kernels with / without PDL, eager and in a graph
(cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_probe launch_probe.cu && ./launch_probe) > gpurun_out/r2bi_launch.log 2>&1
