for i in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_network.py tests/test_gpu_u8.py tests/test_gpu_ops.py -q -x 2>&1 | grep -E "^E   |AssertionError|passed|failed" | head -6; done
