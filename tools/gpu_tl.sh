python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for c in "C5" "C2"; do timeout 300 python tools/timeline.py --config $c --steps 10 2>&1 | head -25; done
timeout 600 python bench.py --no-cpu-baseline --steps 20 2>&1 | tail -2
STR_NO_GRAPH=1 timeout 600 python bench.py --no-cpu-baseline --steps 20 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline --steps 20 --config C3 2>&1 | tail -2
