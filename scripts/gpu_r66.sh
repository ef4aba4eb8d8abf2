# L3 gather through L2 only (cp.async.cg) vs L1-allocating (.ca): two builds
bash scripts/ab_libs.sh "timeout 300 python scripts/frame_probe.py --profile | grep conv_tc_tail | tail -1 | grep -o 'conv_tc_tail.4.=[0-9.]*us'" base.so cg.so
bash scripts/ab_libs.sh "timeout 300 python bench.py --quick --steps 30 --streams 16 2>/dev/null | tail -1 | cut -c1-120" base.so cg.so
