# tail filters as a kernel parameter (constant cache) vs shared memory
for i in 1 2; do for h in 0 1; do echo -n "HEADP=$h "; CBX_TC_HEADP=$h timeout 300 python scripts/frame_probe.py --profile 2>&1 | grep conv_tc_tail | tail -1 | grep -o "conv_tc_tail\[4\]=[0-9.]*us"; done; done
