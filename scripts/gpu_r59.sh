q() { echo -n "$QA : "; timeout 300 python bench.py --quick --steps 30 $QA 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; }
QA="--streams 16" q
QA="--streams 24" q
QA="--streams 32" q
QA="--streams 48" q
QA="--streams 32 --lanes 4" q
