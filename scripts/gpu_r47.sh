timeout 1500 python -m pytest tests/test_gpu_tc.py -q -x -k "groups" 2>&1 | grep -E "^E   |FAILED|passed|failed" | head -8
