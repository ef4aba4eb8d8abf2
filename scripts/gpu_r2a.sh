# r2a: full GPU test suite, smoke, bench (no CPU leg)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader; nproc
timeout 1200 python -m pytest tests -m gpu -q -x -rs --durations=15 2>&1 | tail -60 > gpurun_out/r2a_pytest.log; cat gpurun_out/r2a_pytest.log | tail -40
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; tail -3 gpurun_out/r2a_smoke.log
timeout 600 python bench.py --no-cpu > gpurun_out/r2a_bench.log 2>&1; tail -8 gpurun_out/r2a_bench.log
