python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_rstr.py tests/test_gpu_ksrft.py tests/test_gpu_trals.py tests/test_gpu_edges.py -x -q 2>&1 | tail -2
for i in 1 2; do for pdl in 1 0; do for c in C5 C2 C4; do STR_PDL=$pdl timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/pdl.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/pdl.log').read().strip().splitlines()[-1]);print('pdl $pdl $c', round(d['ms_per_step'],4))"; done; done; done
for pdl in 1 0; do STR_PDL=$pdl timeout 300 python bench.py --config C4 --variant uniform --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/pdl.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/pdl.log').read().strip().splitlines()[-1]);print('pdl $pdl rstr_u', round(d['ms_per_step'],4))"; done
