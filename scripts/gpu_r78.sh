timeout 1200 python -m pytest -x -q tests/test_gpu_tc.py -k "f16" 2>&1 | tail -4
