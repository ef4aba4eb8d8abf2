# layer-3 grid cap (SMs left to the other lane's tensor-core kernels), whole step
q() { echo -n "$QE : "; timeout 300 env $QE python bench.py --quick --steps 30 --streams 16 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; }
for i in 1 2; do QE="CBX_X=0" q; QE="CBX_TC_MAXCTAS_WIDE=140" q; QE="CBX_TC_MAXCTAS_WIDE=132" q; QE="CBX_TC_MAXCTAS_WIDE=124" q; done
