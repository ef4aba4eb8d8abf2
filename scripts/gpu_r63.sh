# CTA pairs with a relaxed (no GPU-scope fence) peer relay, packed fp16 operands
f() { grep total | sed -E 's/(pair=[0-9] stages=[a-z0-9]+).*(conv_tc\[2\]=[0-9.]+).*(conv_tc_tail\[4\]=[0-9.]+).*/\1 \2 \3/'; }
timeout 600 python scripts/tc_probe.py --modes 0,1 --streams 8 --only cbinfer 2>&1 | f
timeout 600 python scripts/tc_probe.py --modes 1 --streams 8 --only cbinfer --stages 3,4,5,6,7 2>&1 | f
timeout 600 python scripts/tc_probe.py --modes 0 --streams 8 --only cbinfer --stages 3,4 2>&1 | f
