python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rstr.py tests/test_gpu_trals.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/plain.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/plain.log').read().strip().splitlines()[-1]); print('graph', d['ms_per_step'], d['roofline']['frac'])"
bash tools/gpu_probe.sh
