# r2j: ncu of the 8-bit path kernels (steady frames, 8 streams, one lane)
mkdir -p gpurun_out
python scripts/frame_probe.py --frames 4 --profile 2>&1 | tail -5
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:detect_rgb8|conv_tc_kernel|dilate_compact|point_" -s 14 -c 12 -o gpurun_out/r2j_u8 python scripts/frame_probe.py --frames 3 > gpurun_out/r2j_ncu.out 2>&1; echo ncu rc=$?; tail -3 gpurun_out/r2j_ncu.out
