mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=25 2>&1 | tail -90 > gpurun_out/r2c_pytest.log; tail -50 gpurun_out/r2c_pytest.log
timeout 600 python -m pytest tests/test_dropin.py -m gpu -q -s -k acceptance 2>&1 | tail -15 > gpurun_out/r2c_accept.log; cat gpurun_out/r2c_accept.log
