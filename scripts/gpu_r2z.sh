mkdir -p gpurun_out
CBX_MPR_F16=1 CBX_MPR_R=1 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:conv_mpr" -s 3 -c 1 -o gpurun_out/r2z_mpr1 python scripts/frame_probe.py --frames 3 > gpurun_out/r2z_ncu.out 2>&1; echo ncu rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:conv_tc" -s 2 -c 1 -o gpurun_out/r2z_l2tc python scripts/frame_probe.py --frames 3 > gpurun_out/r2z_ncu2.out 2>&1; echo ncu rc=$?
