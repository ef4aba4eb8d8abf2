for i in 1 2 3 4 5; do timeout 900 python -m pytest tests/test_gpu_tc.py -q -k mpr 2>&1 | grep -E "^E   |FAILED|passed|failed" | head -6; done
