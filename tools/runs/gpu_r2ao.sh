#!/bin/bash
# factor probe: symmetrisation pass run twice (cold vs warm code)
(cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DFC_PROBE -DFC_SYM2 -I../../include -I../../paper_2307_00719_b200/csrc -o fcs fc_probe.cu && ./fcs 100 && ./fcs 64) > gpurun_out/r2ao_probe.log 2>&1
