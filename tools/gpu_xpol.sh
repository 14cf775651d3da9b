python paper_2307_00719_b200/build.py 2>&1 | tail -1
for x in 0 1 2 0 1; do for c in C5; do
STR_TF_XPOL1=$x timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/xp.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/xp.log').read().strip().splitlines()[-1]);r=d['roofline'];print('xpol $x $c', round(d['ms_per_step'],4), r['pass1_us'], r['pass2_us'], r['frac'], r.get('kernel_span_us'))"
done; done
STR_TF_XPOL1=1 timeout 300 python bench.py --config C4 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/xp.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/xp.log').read().strip().splitlines()[-1]);r=d['roofline'];print('xpol 1 C4', round(d['ms_per_step'],4), r['pass1_us'], r['pass2_us'], r['frac'], r.get('kernel_span_us'))"
