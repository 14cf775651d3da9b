#!/bin/bash
# what-if refresh at HEAD (diagnostic build; masks: 1 factor, 2 tables, 4 passes, 8 absorbs, 16 chain GEMMs, 32 rows, 64 Grams)
bash tools/gpu_whatif2.sh > gpurun_out/r2bn_whatif.log 2>&1
