# usage: bash scripts/gpu_profile.sh TAG   -- ncu launch list + full captures of the hot kernels
TAG=${1:-prof}
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_launches.out 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 6 -c 2 \
  -o gpurun_out/${TAG}_conv_tc $B > gpurun_out/${TAG}_conv_tc.out 2>&1
echo "conv_tc rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"detect_planar|dilate|compact|pool_kernel|conv_exact" -s 12 -c 6 \
  -o gpurun_out/${TAG}_hbm $B > gpurun_out/${TAG}_hbm.out 2>&1
echo "hbm kernels rc=$?"
ls -la gpurun_out/
