#!/bin/bash
# What-if analysis of the C5 / C4 step on a diagnostic build (STR_DBG_SKIP masks):
# 1 factor, 2 tables, 4 contraction passes, 8 absorbs, 16 chain GEMMs, 32 rows solves, 64 Grams
STR_BUILD_DIAG=1 python paper_2307_00719_b200/build.py 2>&1 | tail -1
for c in C5 C4; do
for m in 0 1 2 4 8 16 32 64 17 33 96 113 127; do
  v=$(STR_DBG_SKIP=$m timeout 120 python bench.py --config $c --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,1))")
  echo "$c skip=$m step_us: $v"
done
done
python paper_2307_00719_b200/build.py 2>&1 | tail -1
