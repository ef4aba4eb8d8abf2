TAG=${1:-p9}
mkdir -p gpurun_out
timeout 200 python scripts/tc_probe.py --modes 0 --dbg 0,16,5,21,23,87,80 --only cbinfer --reps 3 > gpurun_out/${TAG}_probe.log 2>&1
grep -o "pair=.*cbinfer\|conv_tc_tail\[4\]=[0-9.]*" gpurun_out/${TAG}_probe.log | paste - -
