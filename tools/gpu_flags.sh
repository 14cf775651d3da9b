python paper_2307_00719_b200/build.py 2>&1 | tail -1
for f in 0 4 32 36 128; do
STR_TF_DBGFLAGS=$f timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/fl.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/fl.log').read().strip().splitlines()[-1]);r=d['roofline'];print('flags $f', round(d['ms_per_step'],4), r['pass1_us'], r['pass2_us'], r.get('kernel_span_us'))"
done
