# L3 bound: no A gather / no epilogue math / neither (timing-only builds; results wrong)
bash scripts/ab_libs.sh "timeout 300 python scripts/frame_probe.py --profile | grep conv_tc_tail | tail -1 | grep -o 'conv_tc_tail.4.=[0-9.]*us'" base.so noa.so noepi.so both.so
