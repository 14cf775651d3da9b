python paper_2307_00719_b200/build.py 2>&1 | tail -1
for f in 0 1 2 3 4 36 128 256 768; do echo "flags $f"; STR_TF_DBGFLAGS=$f timeout 120 python tools/launchcost.py 2>&1 | grep "20 back" ; done
