# What-if analysis of the C5 step: skip kernel classes (STR_DBG_SKIP bitmask) and time the step.
python paper_2307_00719_b200/build.py 2>&1 | tail -1
for m in 0 1 2 4 8 16 32 64 17 49 113 127; do
  v=$(STR_DBG_SKIP=$m timeout 120 python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,1))")
  echo "skip=$m step_us: $v"
done
