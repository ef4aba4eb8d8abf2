TAG=${1:-p3}
mkdir -p gpurun_out
timeout 600 python scripts/tc_probe.py --modes 0 --stages 2,3 --reps 2 > gpurun_out/${TAG}_probe.log 2>&1
timeout 600 python scripts/tc_probe.py --modes 1 --stages 2,3,4,5,6 --reps 2 >> gpurun_out/${TAG}_probe.log 2>&1
grep -o "pair=.*conv_tc\[2\]=[0-9.]*\|conv_tc_tail\[4\]=[0-9.]*" gpurun_out/${TAG}_probe.log
