timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_network.py -q -x 2>&1 | tail -2
python scripts/frame_probe.py --frames 4 --profile 2>&1 | tail -2 | head -1
CBX_TC_NO_XROW=1 python scripts/frame_probe.py --frames 4 --profile 2>&1 | tail -2 | head -1
q() { timeout 300 python bench.py --quick --steps 30 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value']), round(d['ms_per_step'],4), d['lanes'], d['clocks']['sm_mhz'])"; }
q
