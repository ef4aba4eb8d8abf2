timeout 600 python -m pytest tests/test_gpu_u8.py tests/test_gpu_network.py -q -x 2>&1 | tail -3
