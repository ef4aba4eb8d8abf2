# L2 conv bound: no A gather / no compare+store epilogue / B fetched once per CTA (timing-only builds)
bash scripts/ab_libs.sh "timeout 300 python scripts/frame_probe.py --profile | tail -3 | head -1 | grep -o 'conv_tc.2.=[0-9.]*us'" base.so l2noa.so l2noepi.so l2nob.so l2all.so
