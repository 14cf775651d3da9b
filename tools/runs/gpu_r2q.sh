#!/bin/bash
python paper_2307_00719_b200/build.py 2>&1 | tail -1
timeout 300 python tools/timeline.py --config C4 --variant uniform --steps 10 > gpurun_out/r2q.log 2>&1
