# TMEM serialization hypothesis: layer 2 on CUDA cores (conv_exact) so it can co-run with the other lane's layer 3
timeout 300 python scripts/frame_probe.py --profile 2>&1 | tail -3 | head -1
CBX_TC_OFF=2 timeout 300 python scripts/frame_probe.py --profile 2>&1 | tail -3 | head -1
q() { echo -n "$QE : "; timeout 300 env $QE python bench.py --quick --steps 30 --streams 16 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; }
for i in 1 2; do QE="CBX_X=0" q; QE="CBX_TC_OFF=2" q; done
