mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -5 > gpurun_out/r2e_tc.log; cat gpurun_out/r2e_tc.log
for P in f16 tf32; do
timeout 300 python scripts/tc_probe.py --modes 0,1 --precision $P --streams 8 --reps 3 2>&1 | tail -4
done
timeout 300 python scripts/tc_probe.py --modes 1 --precision f16 --streams 8 --reps 3 --stages 3,4,5,6 --only cbinfer 2>&1 | tail -4
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:conv_tc_kernel" -s 12 -c 2 -o gpurun_out/r2e_l3 python scripts/tc_probe.py --modes 0 --precision f16 --streams 8 --reps 1 --only cbinfer > gpurun_out/r2e_ncu.out 2>&1; echo ncu rc=$?; tail -2 gpurun_out/r2e_ncu.out
