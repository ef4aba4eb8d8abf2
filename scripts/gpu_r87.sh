# layer-2 pixel groups (R = 2, two stages) as the default: parity suites, kernel time, step A/B
timeout 1500 python -m pytest -x -q tests -m gpu 2>&1 | tail -3
for e in "CBX_TC_GROUP=1" "CBX_X=0"; do echo -n "$e "; env $e timeout 300 python scripts/frame_probe.py --profile 2>&1 | tail -3 | head -1 | grep -o 'dilate_compact.2.=[0-9.]*us\|conv_tc.2.=[0-9.]*us\|conv_tc_tail.4.=[0-9.]*us' | tr '\n' ' '; echo; done
q() { echo -n "$QE : "; timeout 300 env $QE python bench.py --quick --steps 30 --streams 16 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; }
for i in 1 2 3; do QE="CBX_TC_GROUP=1" q; QE="CBX_X=0" q; done
