python paper_2307_00719_b200/build.py 2>&1 | tail -1
for g in 144 120 132 140 148 144; do
STR_TF_GRID=$g timeout 300 python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/gr.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/gr.log').read().strip().splitlines()[-1]);r=d['roofline'];print('grid $g', round(d['ms_per_step'],4), r['pass1_us'], r['pass2_us'], r['frac'], r.get('kernel_span_us'))"
done
