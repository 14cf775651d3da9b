python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_contract.py tests/test_gpu_stress.py tests/test_gpu_edges.py tests/test_gpu_trals.py -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "C4 or C5_first or C2" 2>&1 | tail -2
for i in 1 2; do for c in C5 C4 C2; do timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/wp.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/wp.log').read().strip().splitlines()[-1]);r=d['roofline'];print('$c', round(d['ms_per_step'],4), r['pass1_us'], r['pass2_us'], r['frac'], r.get('kernel_span_us'))"; done; done
