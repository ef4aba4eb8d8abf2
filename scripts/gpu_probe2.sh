# usage: bash scripts/gpu_probe2.sh TAG -- bounded tc tests + timing probe of the tcgen05 modes
TAG=${1:-p2}
mkdir -p gpurun_out
timeout 180 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -5 > gpurun_out/${TAG}_tc.log; cat gpurun_out/${TAG}_tc.log
timeout 300 python scripts/tc_probe.py --modes 0,1 > gpurun_out/${TAG}_probe.log 2>&1; grep pair= gpurun_out/${TAG}_probe.log
