python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_ksrft.py tests/test_gpu_rstr.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --config C4 --variant ksrft --steps 20 --warmup 5 --e2e-steps 5 > gpurun_out/bench_rstr_k.log 2>&1; tail -c 1500 gpurun_out/bench_rstr_k.log
