python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_contract.py tests/test_gpu_stress.py tests/test_gpu_edges.py -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "C4 or C2 or C5_first" 2>&1 | tail -2
for c in C4 C2 C5; do echo "$c"; timeout 120 python tools/launchcost.py $c 2>&1 | grep "20 back"; done
for c in C4 C2 C5; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/na.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/na.log').read().strip().splitlines()[-1]);r=d['roofline'];print('$c', round(d['ms_per_step'],4), r['pass1_us'], r['pass2_us'], r['frac'])"; done
