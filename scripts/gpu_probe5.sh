TAG=${1:-p8}
mkdir -p gpurun_out
timeout 200 python scripts/tc_probe.py --modes 0,1 --dbg 0,1,4,5,7,16,23 --only baseline --reps 2 > gpurun_out/${TAG}_probe.log 2>&1
grep -o "pair=.*baseline\|conv_tc_tail\[4\]=[0-9.]*" gpurun_out/${TAG}_probe.log | paste - -
