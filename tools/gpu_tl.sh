python paper_2307_00719_b200/build.py 2>&1 | tail -1
for g in 148 144 143 140; do
  STR_TF_GRID=$g timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/plain_g$g.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/plain_g$g.log').read().strip().splitlines()[-1]); print($g, d['ms_per_step'], d['roofline']['frac'], d['roofline']['pass1_us'], d['roofline']['pass2_us'], d['roofline'].get('kernel_span_us'))"
done
