python paper_2307_00719_b200/build.py 2>&1 | tail -1
for c in C4 C2; do for f in 0 3 256; do echo "$c flags $f"; STR_TF_DBGFLAGS=$f timeout 120 python tools/launchcost.py $c 2>&1 | grep "20 back"; done; done
