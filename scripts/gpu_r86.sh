# lane stream priorities (lane 0 high): whole step
q() { echo -n "$QE : "; timeout 300 env $QE python bench.py --quick --steps 30 --streams 16 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; }
for i in 1 2; do QE="CBX_LANE_PRIO=0" q; QE="CBX_LANE_PRIO=1" q; done
