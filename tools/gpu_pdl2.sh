python paper_2307_00719_b200/build.py 2>&1 | tail -1
for i in 1 2; do for m in 0 1 3 5 7; do for c in C5 C4; do STR_PDL=$m timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/pdl.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/pdl.log').read().strip().splitlines()[-1]);print('mask $m $c', round(d['ms_per_step'],4))"; done; done; done
