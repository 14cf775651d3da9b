python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_contract.py tests/test_gpu_edges.py tests/test_gpu_trals.py -x -q 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "C3 or f64" 2>&1 | tail -2
for a in "--config C3" "--contract f64"; do timeout 300 python bench.py $a --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/f64b.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/f64b.log').read().strip().splitlines()[-1]);r=d['roofline'];print('$a', round(d['ms_per_step'],4), r['pass1_us'], r['pass2_us'], r['frac'])"; done
