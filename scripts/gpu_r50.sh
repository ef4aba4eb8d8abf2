q() { echo -n "$* : "; env "$@" timeout 300 python bench.py --quick --steps 30 $QA 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; }
for i in 1 2; do q CBX_STAGGER=0; q CBX_STAGGER=1; done
QA="--lanes 3" q CBX_STAGGER=1
QA="--lanes 4" q CBX_STAGGER=1
