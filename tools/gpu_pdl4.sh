python paper_2307_00719_b200/build.py 2>&1 | tail -1
STR_PDL=29 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -x -q 2>&1 | tail -2
for i in 1 2; do for m in 13 29; do for c in C5 C4 C2; do STR_PDL=$m timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/pdl.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/pdl.log').read().strip().splitlines()[-1]);print('mask $m $c', round(d['ms_per_step'],4))"; done; done; done
