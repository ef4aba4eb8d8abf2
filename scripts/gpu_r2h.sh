# r2h: session-2 baseline: full GPU tests, smoke, default bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader; nproc
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/r2h_pytest.log 2>&1; tail -25 gpurun_out/r2h_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; tail -3 gpurun_out/r2h_smoke.log
timeout 900 python bench.py > gpurun_out/r2h_bench.log 2>&1; tail -3 gpurun_out/r2h_bench.log
