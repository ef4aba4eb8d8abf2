# layer 1 on IDP4A (no TMEM): parity, kernel time, two-lane step A/B
timeout 900 python -m pytest -x -q tests/test_gpu_u8.py tests/test_gpu_network.py tests/test_gpu_benchconfig.py 2>&1 | tail -3
for d in 0 1; do echo -n "DP4A=$d "; CBX_L1_DP4A=$d timeout 300 python scripts/frame_probe.py --profile 2>&1 | tail -3 | head -1 | cut -c1-300; done
q() { echo -n "$QE : "; timeout 300 env $QE python bench.py --quick --steps 30 --streams 16 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; }
for i in 1 2; do QE="CBX_L1_DP4A=0" q; QE="CBX_L1_DP4A=1" q; done
