mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=20 2>&1 | tail -80 > gpurun_out/r2b_pytest.log; tail -45 gpurun_out/r2b_pytest.log
