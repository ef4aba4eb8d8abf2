timeout 1500 python -m pytest tests/test_gpu_u8.py -q -x 2>&1 | grep -E "^E   |FAILED|passed|failed" | head -5
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed -k "regex:detect_rgb8" -s 2 -c 1 python scripts/frame_probe.py --frames 3 2>&1 | grep -E "duration|inst_executed|throughput" | head
q() { echo -n "$* : "; env "$@" timeout 300 python bench.py --quick --steps 30 $QA 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"; }
q CBX_X=0
q CBX_X=0
