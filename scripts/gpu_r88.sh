# layer 2 on kind::f16 (packed shadow, pixel groups): per-layer bound, kernel time, step A/B
timeout 900 python -m pytest -x -q tests/test_gpu_l2f16.py 2>&1 | tail -4
for e in "CBX_X=0" "CBX_L2_F16=1"; do echo -n "$e "; env $e timeout 300 python scripts/frame_probe.py --profile 2>&1 | tail -3 | tr '\n' ' ' | grep -o 'pool.1.=[0-9.]*us\|dilate_compact.2.=[0-9.]*us\|conv_tc.2.=[0-9.]*us\|conv_tc_tail.4.=[0-9.]*us\|L3: \[.*\]' | tr '\n' ' '; echo; done
q() { echo -n "$QE : "; timeout 300 env $QE python bench.py --quick --steps 30 --streams 16 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; }
for i in 1 2 3; do QE="CBX_X=0" q; QE="CBX_L2_F16=1" q; done
