# L3 launch bounds: minBlocks 1 for the fused-tail kernel (no spills) vs 2
bash scripts/ab_libs.sh "timeout 300 python scripts/frame_probe.py --profile | grep conv_tc_tail | tail -1 | grep -o 'conv_tc_tail.4.=[0-9.]*us'" base.so lb1.so
bash scripts/ab_libs.sh "timeout 300 python bench.py --quick --steps 30 --streams 16 2>/dev/null | tail -1 | cut -c1-100" base.so lb1.so
