# usage: bash scripts/gpu_quick.sh TAG [bench args...] -- tc tests (bounded), gpu tests, short bench
TAG=${1:-q}; shift
mkdir -p gpurun_out
timeout 180 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -25 > gpurun_out/${TAG}_tc.log; cat gpurun_out/${TAG}_tc.log
if grep -q "passed" gpurun_out/${TAG}_tc.log && ! grep -q "failed\|error" gpurun_out/${TAG}_tc.log; then
  timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_pytest.log
  timeout 300 python bench.py --no-cpu "$@" > gpurun_out/${TAG}_bench.log 2>&1; tail -5 gpurun_out/${TAG}_bench.log
fi
