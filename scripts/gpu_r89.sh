# layer-2 group epilogue: prefetch the stored values (L2 / L1) while the MMAs run
bash scripts/ab_libs.sh "timeout 300 python scripts/frame_probe.py --profile | tail -3 | head -1 | grep -o 'conv_tc.2.=[0-9.]*us\|conv_tc_tail.4.=[0-9.]*us' | tr '\n' ' '; echo" base.so gpf2.so gpf1.so
bash scripts/ab_libs.sh "timeout 300 python bench.py --quick --steps 30 --streams 16 2>/dev/null | tail -1 | cut -c1-90" base.so gpf2.so gpf1.so
