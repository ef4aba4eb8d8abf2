mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_network.py tests/test_gpu_u8.py tests/test_gpu_ops.py -q -x 2>&1 | tail -3
python scripts/frame_probe.py --frames 4 --profile 2>&1 | tail -3
