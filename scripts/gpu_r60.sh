# packed fp16 layer-3 input: parity, then A/B against the padded layout
timeout 900 python -m pytest -x -q tests/test_gpu_tc.py tests/test_gpu_network.py tests/test_gpu_u8.py tests/test_gpu_benchconfig.py 2>&1 | tail -5
q() { echo -n "$QA : "; timeout 300 env $QE python bench.py --quick --steps 30 $QA 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; }
for i in 1 2; do
QE="CBX_TC_PACK=0" QA="--streams 16" q
QE="CBX_TC_PACK=1" QA="--streams 16" q
done
CBX_TC_PACK=0 timeout 300 python scripts/frame_probe.py --profile 2>&1 | tail -14
CBX_TC_PACK=1 timeout 300 python scripts/frame_probe.py --profile 2>&1 | tail -14
