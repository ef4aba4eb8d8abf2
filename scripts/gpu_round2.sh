# round-2 evidence: default bench (as the driver runs it), reference arm, ncu launch list + steady-frame capture
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader; nproc
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-400
B="python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --no-cudnn --streams 16"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 300 --csv \
  --log-file gpurun_out/${TAG}_launches.csv $B > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"detect|dilate|conv|point" -s 12 -c 10 -o gpurun_out/${TAG}_frame $B > gpurun_out/${TAG}_frame.out 2>&1; echo "frame capture rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${TAG}_ref.log 2>&1; tail -1 gpurun_out/${TAG}_ref.log | cut -c1-300
