python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 1500 python tools/compare_sweeps.py --set order --methods "STR,rSTR-U,rSTR-K" --out gpurun_out/compare_k_order.json 2>&1 | tail -6
timeout 900 python tools/compare_sweeps.py --set rank --methods "STR,rSTR-U,rSTR-K" --out gpurun_out/compare_k_rank.json 2>&1 | tail -4
