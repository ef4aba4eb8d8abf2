# tcgen05.fence::after_thread_sync per K-block: cost (timing builds)
bash scripts/ab_libs.sh "timeout 300 python scripts/frame_probe.py --profile | tail -3 | head -1 | grep -o 'conv_tc.2.=[0-9.]*us\|conv_tc_tail.4.=[0-9.]*us' | tr '\n' ' '; echo" base.so nof.so l2all.so l2allnof.so
