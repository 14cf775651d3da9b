python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_ksrft.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --config C4 --variant ksrft --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ks_bench.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/ks_bench.log').read().strip().splitlines()[-1]);print('ksrft C4 ms/step',d['ms_per_step'], d['roofline'].get('mix_us'), d['roofline'].get('frac'))"
python tools/ks_probe.py C4 1 && ncu --clock-control none -k "regex:k_mix_(pq|mode)" --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size --csv python tools/ks_probe.py C4 1 > gpurun_out/ks_ncu.csv 2>&1
