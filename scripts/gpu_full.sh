# usage: bash scripts/gpu_full.sh TAG -- tests, default bench (incl. CPU baseline, e2e), ncu launch list + captures
TAG=${1:-full}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-300
B="python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --streams ${STREAMS:-16}"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --cache-control none -c 300 --csv \
  --log-file gpurun_out/${TAG}_launches.csv $B > /dev/null 2>&1; echo "launches rc=$?"
# steady frame 1 of lane 0: skip both lanes' full first frames (2 x 5 launches), then 11 launches
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"detect|dilate|conv|point" -s ${SKIP:-10} -c 11 -o gpurun_out/${TAG}_frame $B > gpurun_out/${TAG}_frame.out 2>&1; echo "frame capture rc=$?"
