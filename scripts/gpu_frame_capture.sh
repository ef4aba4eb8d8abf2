TAG=${1:-frame}
B="python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --streams ${STREAMS:-16}"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"detect|dilate|conv|point" -s ${SKIP:-10} -c 11 -o gpurun_out/${TAG}_frame $B > gpurun_out/${TAG}_frame.out 2>&1; echo "frame capture rc=$?"
