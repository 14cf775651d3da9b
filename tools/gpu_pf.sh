python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_contract.py -x -q 2>&1 | tail -2
for pf in 1 0 1 0; do for c in C5 C4; do
STR_TF_PREFETCH=$pf timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/pf.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/pf.log').read().strip().splitlines()[-1]);r=d['roofline'];print('pf $pf $c', round(d['ms_per_step'],4), r['pass1_us'], r['pass2_us'], r['frac'], r.get('kernel_span_us'))"
done; done
