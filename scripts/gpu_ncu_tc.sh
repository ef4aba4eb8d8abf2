# usage: bash scripts/gpu_ncu_tc.sh TAG MODES ENGINE -- ncu --set full of the first L3 (tail) conv_tc launch per mode
TAG=${1:-ncutc}; MODES=${2:-0,1}; ENG=${3:-baseline}
mkdir -p gpurun_out
for m in ${MODES//,/ }; do
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:conv_tc_kernel.*8, " -c 1 \
  -o gpurun_out/${TAG}_m${m} python scripts/tc_probe.py --modes ${m} --only ${ENG} --reps 1 > gpurun_out/${TAG}_m${m}_ncu.out 2>&1
echo "ncu m${m} rc=$?"; tail -1 gpurun_out/${TAG}_m${m}_ncu.out
done
