python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in "C5" "C2" "C3"; do timeout 300 python tools/timeline.py --config $c --steps 10 2>&1 | head -25; done
