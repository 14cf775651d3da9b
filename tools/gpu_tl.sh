python paper_2307_00719_b200/build.py 2>&1 | tail -1
echo "== graph"; timeout 300 python tools/c5_debug.py C5 2>&1 | tail -6
echo "== eager"; STR_NO_GRAPH=1 timeout 300 python tools/c5_debug.py C5 2>&1 | tail -6
echo "== f64"; timeout 300 python tools/c5_debug.py C5 f64 4 2>&1 | tail -6
