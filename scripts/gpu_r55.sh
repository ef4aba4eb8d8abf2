timeout 1500 python -m pytest tests/test_gpu_network.py tests/test_gpu_u8.py tests/test_gpu_ops.py -q 2>&1 | tail -1
q() { echo -n "$* : "; env "$@" timeout 300 python bench.py --quick --steps 40 $QA 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; }
for i in 1 2 3 4; do q CBX_X=0; done
