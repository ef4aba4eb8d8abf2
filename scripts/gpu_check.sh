set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g | head -2
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r1_pytest.log
cat gpurun_out/r1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1; tail -5 gpurun_out/r1_smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r1_bench.log 2>&1; tail -5 gpurun_out/r1_bench.log
