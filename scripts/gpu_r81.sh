# layer-2 pixel groups (R adjacent pixels per tensor-core row) vs one pixel per row, whole step
q() { echo -n "$QE : "; timeout 300 env $QE python bench.py --quick --steps 30 --streams 16 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; }
for i in 1 2; do QE="CBX_TC_GROUP=1" q; QE="CBX_TC_GROUP=2" q; QE="CBX_TC_GROUP=4" q; done
for g in 1 2 4; do echo -n "G=$g "; CBX_TC_GROUP=$g timeout 300 python scripts/frame_probe.py --profile 2>&1 | tail -3 | head -1 | grep -o 'dilate_compact.2.=[0-9.]*us\|conv_tc.2.=[0-9.]*us' | tr '\n' ' '; echo; done
