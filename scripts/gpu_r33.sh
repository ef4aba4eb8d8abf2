timeout 900 python -m pytest tests/test_gpu_u8.py -q -x 2>&1 | grep -E "^E |FAILED|passed|failed|Error" | head -12
