# change-rate sweep at 1080p (the metric's x-axis): frames/s and speedup over dense per recipe
timeout 1200 python bench.py --sweep --no-cpu --no-e2e > gpurun_out/r2b_sweep.log 2>&1; tail -1 gpurun_out/r2b_sweep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d.get('sweep')))"
