python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_ksrft.py -x -q 2>&1 | tail -15
timeout 300 python bench.py --config C4 --variant ksrft --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ks_bench.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/ks_bench.log').read().strip().splitlines()[-1]);print('ksrft C4 ms/step',d['ms_per_step'])"
timeout 300 python tools/timeline.py --config C4 --variant ksrft --steps 10 2>&1 | head -30
