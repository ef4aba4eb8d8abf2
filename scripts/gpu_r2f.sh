mkdir -p gpurun_out
P="python scripts/tc_probe.py --precision f16 --streams 8 --reps 1 --only cbinfer"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:conv_tc_kernel" -s 4 -c 2 -o gpurun_out/r2f_tc_single $P --modes 0 > gpurun_out/r2f_tc_single.out 2>&1; echo "single rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:conv_tc_kernel" -s 4 -c 2 -o gpurun_out/r2f_tc_pair $P --modes 1 > gpurun_out/r2f_tc_pair.out 2>&1; echo "pair rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:dilate_compact|detect_c3|point_work|conv_planar" -s 8 -c 8 -o gpurun_out/r2f_masks $P --modes 0 > gpurun_out/r2f_masks.out 2>&1; echo "masks rc=$?"
ls -la gpurun_out/*.ncu-rep
