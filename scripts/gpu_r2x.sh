q() { timeout 300 python bench.py --quick --steps 30 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value']), round(d['ms_per_step'],4), d['lanes'], d['clocks']['sm_mhz'])"; }
q
CBX_TC_STAGES=3 q
q --lanes 3
q --lanes 4
q --streams 24 --lanes 3
q --streams 32 --lanes 4
q --streams 32 --lanes 2
q --streams 8 --lanes 1
