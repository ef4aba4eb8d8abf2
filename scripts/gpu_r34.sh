for i in 1 2 3 4 5 6; do timeout 900 python -m pytest tests/test_gpu_u8.py tests/test_gpu_network.py -q 2>&1 | grep -E "^E   |FAILED|passed|failed" | head -8; done
