# L3 bound with CTA pairs (relaxed relay): no A gather / no epilogue math / neither (timing-only builds)
f() { grep total | sed -E 's/(pair=[0-9] stages=[a-z0-9]+).*(conv_tc_tail\[4\]=[0-9.]+).*/\1 \2/'; }
bash scripts/ab_libs.sh "timeout 300 python scripts/tc_probe.py --modes 1 --streams 8 --only cbinfer | grep total | grep -o 'conv_tc_tail.4.=[0-9.]*'" pbase.so pnoa.so pnoepi.so pboth.so
