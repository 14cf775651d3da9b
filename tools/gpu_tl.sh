python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_rstr.py -x -q 2>&1 | tail -4
STR_RSTR_HOST_DRAWS=1 timeout 900 python -m pytest tests/test_gpu_rstr.py -x -q 2>&1 | tail -2
for v in uniform leverage; do
timeout 300 python bench.py --config C4 --variant $v --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/plain_$v.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/plain_$v.log').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['value'], d['gpu_launches'])" || tail -5 gpurun_out/plain_$v.log
done
