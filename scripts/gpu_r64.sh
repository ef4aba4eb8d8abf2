# ncu --set full of a steady L3 launch, single CTA vs CTA pair
mkdir -p gpurun_out
for m in 0 1; do
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:conv_tc_kernel.*8, " -s 3 -c 1 \
  -o gpurun_out/r64_m${m} python scripts/tc_probe.py --modes ${m} --only cbinfer --reps 1 --streams 8 > gpurun_out/r64_m${m}.out 2>&1
echo "ncu m${m} rc=$?"
done
