#!/bin/bash
(cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DFC_PROBE -I../../include -I../../paper_2307_00719_b200/csrc -o fc_probe fc_probe.cu && ./fc_probe 100) > gpurun_out/r2n_probe.log 2>&1
python paper_2307_00719_b200/build.py 2>&1 | tail -1
for env in "STR_GF=1" "STR_GF=0"; do
  echo "== $env"
  env $env timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C5 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,1), d['roofline']['pass1_us'], d['roofline']['pass2_us'])"
done >> gpurun_out/r2n_probe.log 2>&1
