mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_network.py tests/test_gpu_benchconfig.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -5
timeout 600 python bench.py --no-cpu --no-cudnn > gpurun_out/r2g_bench.log 2>&1; grep "^\[gpu\]" gpurun_out/r2g_bench.log; tail -1 gpurun_out/r2g_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['per_kernel_ms'], d['e2e']['value'], d['clocks'])"
