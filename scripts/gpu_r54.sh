timeout 1500 python -m pytest tests/test_gpu_network.py tests/test_gpu_u8.py tests/test_gpu_ops.py -q -x 2>&1 | grep -E "^E   |FAILED|passed|failed" | head -5
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum -k "regex:point_work|dilate_compact" -s 3 -c 4 python scripts/frame_probe.py --frames 3 2>&1 | grep -E "point_work|dilate_compact|duration" | head -12
q() { echo -n "$* : "; env "$@" timeout 300 python bench.py --quick --steps 30 $QA 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; }
q CBX_X=0
q CBX_X=0
