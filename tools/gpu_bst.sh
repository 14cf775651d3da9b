python paper_2307_00719_b200/build.py 2>&1 | tail -1
for b in 2 3 4; do for c in C5 C4; do
STR_TF_BSTAGES=$b timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bst.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bst.log').read().strip().splitlines()[-1]);r=d['roofline'];print('bst $b $c', round(d['ms_per_step'],4), r['pass1_us'], r['pass2_us'], r['frac'], r.get('kernel_span_us'))"
done; done
