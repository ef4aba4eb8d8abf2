q() { echo -n "$* : "; env "$@" timeout 300 python bench.py --quick --steps 30 $QA 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; }
q CBX_X=0
q CBX_TC_CTAS_PER_SM=1
QA="--lanes 3" q CBX_X=0
QA="--lanes 4" q CBX_X=0
QA="--lanes 4 --streams 32" q CBX_X=0
QA="--lanes 2 --streams 32" q CBX_X=0
