python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python tools/compare_sweeps.py --set length --methods "STR,rSTR-U,rSTR-K" --out gpurun_out/compare_k_length.json 2>&1 | tail -4
timeout 900 python tools/compare_sweeps.py --set slice --methods "STR,rSTR-U,rSTR-K" --out gpurun_out/compare_k_slice.json 2>&1 | tail -4
