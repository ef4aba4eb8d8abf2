# single-thread MMA issue loop (no per-K-block elect/syncwarp/whole-warp waits): timing
bash scripts/ab_libs.sh "timeout 300 python scripts/frame_probe.py --profile | tail -3 | head -1 | grep -o 'conv_tc.2.=[0-9.]*us\|conv_tc_tail.4.=[0-9.]*us' | tr '\n' ' '; echo" base.so solo.so
bash scripts/ab_libs.sh "timeout 300 python bench.py --quick --steps 30 --streams 16 2>/dev/null | tail -1 | cut -c1-90" base.so solo.so
