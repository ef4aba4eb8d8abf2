# r2i: 8-bit native path (byte detection + kind::i8 layer 1): tests + bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_u8.py -q -x 2>&1 | tail -30 > gpurun_out/r2i_u8.log; cat gpurun_out/r2i_u8.log
timeout 900 python -m pytest tests/test_gpu_network.py -q -x 2>&1 | tail -5
timeout 600 python bench.py --no-cpu --no-cudnn --steps 20 > gpurun_out/r2i_bench.log 2>&1; grep "^\[gpu\]" gpurun_out/r2i_bench.log; tail -1 gpurun_out/r2i_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config']['f32_frames_value'], d['roofline']['frac'], d['roofline']['per_kernel_ms'], d['e2e']['value'], d['config']['speedup_vs_dense'])"
