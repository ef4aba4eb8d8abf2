TAG=${1:-p4}
mkdir -p gpurun_out
timeout 150 python scripts/tc_probe.py --modes 0 --dbg 0,31,95,87,80,64 --only baseline --reps 2 > gpurun_out/${TAG}_probe.log 2>&1
grep -o "pair=.*baseline\|conv_tc_tail\[4\]=[0-9.]*" gpurun_out/${TAG}_probe.log | paste - -
