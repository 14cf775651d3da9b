#!/bin/bash
# chain stream at the highest priority with per-node priorities in the step graph (STR_CHAIN_PRIO=1) vs default
python paper_2307_00719_b200/build.py 2>&1 | tail -1
for p in 0 1 0 1; do
  for c in C5 C4 C3 C2; do
    STR_CHAIN_PRIO=$p timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('prio=$p $c', round(d['ms_per_step'],4), d['roofline'].get('pass1_us'), d['roofline'].get('pass2_us'))" >> gpurun_out/prio.log 2>&1
  done
  STR_CHAIN_PRIO=$p timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant uniform 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('prio=$p C4 rSTR-U', round(d['ms_per_step'],4))" >> gpurun_out/prio.log 2>&1
done
STR_CHAIN_PRIO=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rstr.py -m gpu -q -x -p no:cacheprovider > gpurun_out/prio_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/prio_pytest.log
