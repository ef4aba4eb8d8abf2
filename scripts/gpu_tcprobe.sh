# usage: bash scripts/gpu_tcprobe.sh TAG -- timing probe of the tcgen05 modes + ncu full capture of steady conv_tc launches
TAG=${1:-tcp}
mkdir -p gpurun_out
timeout 300 python scripts/tc_probe.py --modes 0,1 > gpurun_out/${TAG}_probe.log 2>&1; cat gpurun_out/${TAG}_probe.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -c 40 \
  -o gpurun_out/${TAG}_conv_tc python scripts/tc_probe.py --modes 0,1 --only cbinfer --reps 1 > gpurun_out/${TAG}_ncu.out 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${TAG}_ncu.out
