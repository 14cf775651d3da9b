#!/bin/bash
python paper_2307_00719_b200/build.py 2>&1 | tail -1
for env in "STR_GF=1" "STR_GF=0" "STR_GF=1 STR_TF_GRID=140" "STR_GF=0 STR_TF_GRID=146"; do
  echo "== $env"
  env $env timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C5 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,1), d['roofline']['pass1_us'], d['roofline']['pass2_us'])"
done > gpurun_out/r2m.log 2>&1
for env in "STR_GF=1" "STR_GF=0"; do echo "== timeline $env"; env $env timeout 300 python tools/timeline.py --config C5 --steps 10; done >> gpurun_out/r2m.log 2>&1
