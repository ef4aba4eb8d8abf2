mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=30 > gpurun_out/r2d_pytest.log 2>&1; grep -E "^(PASSED|FAILED|ERROR)|passed|failed" gpurun_out/r2d_pytest.log | tail -130
timeout 600 ./tests/dropin/_build/acceptance > gpurun_out/r2d_accept.log 2>&1; cat gpurun_out/r2d_accept.log
