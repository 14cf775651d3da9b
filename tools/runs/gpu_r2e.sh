#!/bin/bash
python paper_2307_00719_b200/build.py 2>&1 | tail -1
for env in "STR_PDL=13" "STR_PDL=0" "STR_INV=0" "STR_PDL=0 STR_INV=0"; do
  echo "== $env"; env $env timeout 300 python tools/loopback_stress.py 2>&1 | grep -E "ok|FAIL|Error"
done > gpurun_out/r2e_stress.log 2>&1
