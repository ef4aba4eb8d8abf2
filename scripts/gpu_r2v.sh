mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_u8.py -q -x -k "test_native_u8_layer1" 2>&1 | grep -E "Error|assert|err|^E " | head -20
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:dilate_compact|point_" -s 8 -c 8 -o gpurun_out/r2v_masks python scripts/frame_probe.py --frames 3 > gpurun_out/r2v_ncu.out 2>&1; echo ncu rc=$?
