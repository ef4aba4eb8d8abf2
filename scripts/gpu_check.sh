# usage: bash scripts/gpu_check.sh TAG [bench args...]
TAG=${1:-run}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 240 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -25 > gpurun_out/${TAG}_tc.log; cat gpurun_out/${TAG}_tc.log
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -3 gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py "$@" > gpurun_out/${TAG}_bench.log 2>&1; tail -6 gpurun_out/${TAG}_bench.log
