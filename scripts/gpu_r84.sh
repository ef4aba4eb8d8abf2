# layer-2 pixel groups (N = 128 costs what N = 64 does) with a smaller footprint
q() { echo -n "$QE : "; timeout 300 env $QE python bench.py --quick --steps 30 --streams 16 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; }
for i in 1 2; do QE="CBX_X=0" q; QE="CBX_TC_GROUP=2 CBX_TC_STAGES=2 CBX_TC_STAGES_WIDE=3" q; QE="CBX_TC_GROUP=2" q; done
for e in "CBX_X=0" "CBX_TC_GROUP=2 CBX_TC_STAGES=2 CBX_TC_STAGES_WIDE=3"; do echo -n "$e "; env $e timeout 300 python scripts/frame_probe.py --profile 2>&1 | tail -3 | head -1 | grep -o 'conv_tc.2.=[0-9.]*us\|conv_tc_tail.4.=[0-9.]*us' | tr '\n' ' '; echo; done
