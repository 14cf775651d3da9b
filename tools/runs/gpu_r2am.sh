#!/bin/bash
# factor what-if probes: 0 normal, 1 no trailing update / V rows, 2 no pivot-block factorization, 3 neither
(cd tools/micro && for w in 0 1 2 3; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DFC_PROBE -DFC_WHATIF=$w -I../../include -I../../paper_2307_00719_b200/csrc -o fcw_$w fc_probe.cu && echo "== whatif $w" && ./fcw_$w 100 && ./fcw_$w 64; done) > gpurun_out/r2am_probe.log 2>&1
