python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_rstr.py tests/test_gpu_ksrft.py -x -q 2>&1 | tail -2
for v in uniform leverage ksrft; do timeout 300 python bench.py --config C4 --variant $v --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/rb_$v.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/rb_$v.log').read().strip().splitlines()[-1]);print('$v', d['ms_per_step'])"; done
python tools/ks_probe.py C4 3 uniform && ncu --clock-control none --metrics gpu__time_duration.sum --csv python tools/ks_probe.py C4 3 uniform > gpurun_out/ru_launches.csv 2>&1
