python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_contract.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for f in 0; do echo flags $f; STR_TF_DBGFLAGS=$f timeout 120 python tools/tftrace.py C5 1 2>/dev/null | head -7; done
timeout 600 python bench.py --no-cpu-baseline --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline'])"
