mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -6 > gpurun_out/r2s_pytest.log; cat gpurun_out/r2s_pytest.log
timeout 900 python bench.py --no-cpu --no-cudnn > gpurun_out/r2s_bench.log 2>&1; grep "^\[gpu\]" gpurun_out/r2s_bench.log; tail -1 gpurun_out/r2s_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config']['f32_frames_value'], d['roofline']['frac'], d['roofline']['per_kernel_ms'], d['e2e']['value'], d['config']['speedup_vs_dense'])"
