TAG=${1:-p11}
mkdir -p gpurun_out
timeout 180 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -3
timeout 200 python scripts/tc_probe.py --modes 0 --reps 3 > gpurun_out/${TAG}_probe.log 2>&1
grep -o "pair=.*\(cbinfer\|baseline\)\|conv_tc\[2\]=[0-9.]*\|conv_tc_tail\[4\]=[0-9.]*" gpurun_out/${TAG}_probe.log | paste - - -
