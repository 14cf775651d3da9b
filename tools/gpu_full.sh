python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_stress.py -q 2>&1 | tail -3 > gpurun_out/stress.log
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 600 python bench.py --contract f64 --no-cpu-baseline > gpurun_out/bench_f64.log 2>&1
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
timeout 600 python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
timeout 600 python bench.py --config C4 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
timeout 600 python bench.py --config C4 --variant uniform --no-cpu-baseline > gpurun_out/bench_rstr_u.log 2>&1
timeout 600 python bench.py --config C4 --variant leverage --no-cpu-baseline > gpurun_out/bench_rstr_l.log 2>&1
timeout 600 python bench.py --config C4 --variant ksrft > gpurun_out/bench_rstr_k.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_mix_(pq|mode)" -s 4 -c 4 -o gpurun_out/prof_ksrft_mix python tools/ks_probe.py C4 2 > gpurun_out/ncu3.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_contract_tf32 -s 6 -c 2 -o gpurun_out/prof_tf32_final $CMD > gpurun_out/ncu2.log 2>&1
echo done
