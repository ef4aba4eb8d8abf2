# r2k: 8-bit path after fast division / conflict-free i8 gather / warp-uniform detect
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_u8.py -q -x 2>&1 | tail -4
python scripts/frame_probe.py --frames 4 --profile 2>&1 | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:detect_rgb8|conv_tc_kernel" -s 5 -c 4 -o gpurun_out/r2k_u8 python scripts/frame_probe.py --frames 3 > gpurun_out/r2k_ncu.out 2>&1; echo ncu rc=$?
