mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -12 > gpurun_out/r2t_pytest.log; cat gpurun_out/r2t_pytest.log
