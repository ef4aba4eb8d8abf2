q() { echo -n "$* : "; env "$@" timeout 300 python bench.py --quick --steps 30 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; }
q CBX_X=0
q CBX_TC_STAGES=3
q CBX_TC_STAGES=3 CBX_MPR_STAGES=2
q CBX_TC_STAGES=3 CBX_MPR_STAGES=3
q CBX_MPR_STAGES=3
q CBX_TC_STAGES=2
q CBX_X=0
