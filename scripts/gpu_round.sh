# usage: bash scripts/gpu_round.sh TAG  -- tests + full default bench (with CPU baseline) + reference arm
TAG=${1:-round}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; tail -8 gpurun_out/${TAG}_bench.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${TAG}_ref.log 2>&1; tail -4 gpurun_out/${TAG}_ref.log
