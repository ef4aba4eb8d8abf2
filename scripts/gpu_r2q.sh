mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_tc.py -q -x -k mpr 2>&1 | tail -4
python scripts/frame_probe.py --frames 4 --profile 2>&1 | tail -3
python scripts/frame_probe.py --frames 2 --profile --engine baseline 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:conv_mpr" -s 2 -c 2 -o gpurun_out/r2q_mpr python scripts/frame_probe.py --frames 3 > gpurun_out/r2q_ncu.out 2>&1; echo ncu rc=$?
