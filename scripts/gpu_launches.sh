# usage: bash scripts/gpu_launches.sh TAG [regex]  -- ncu launch list (+ optional full capture of kernels matching regex)
TAG=${1:-l}; RX=${2:-}
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --streams ${STREAMS:-16}"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --cache-control none -c 300 --csv \
  --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_launches.out 2>&1
echo "launch list rc=$?"
if [ -n "$RX" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 20 -c 8 \
  -o gpurun_out/${TAG}_full $B > gpurun_out/${TAG}_full.out 2>&1
echo "full rc=$?"
fi
