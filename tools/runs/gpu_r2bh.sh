#!/bin/bash
# round-2 final evidence (two-CTA factor): full GPU suite, smoke, benches (all configs / variants), reference arm, ncu launch list + --set full of the contraction
python paper_2307_00719_b200/build.py 2>&1 | tail -1
nvidia-smi -L
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1
for c in C4 C3 C2; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config $c > gpurun_out/bench_${c,,}.log 2>&1; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C5 --contract f64 > gpurun_out/bench_f64.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant uniform > gpurun_out/bench_rstr_u.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant leverage > gpurun_out/bench_rstr_l.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 --config C4 --variant ksrft > gpurun_out/bench_rstr_k.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_contract_tf32 -s 6 -c 2 -o gpurun_out/prof_tf32_final $CMD > gpurun_out/ncu2.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
