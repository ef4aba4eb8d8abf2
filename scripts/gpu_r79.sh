# split accumulator: second-instruction MMAs first while the epilogue drains the shared columns
cp paper_1704_04313_b200/_lib_alt/defer.so paper_1704_04313_b200/_lib/libcbx.so
timeout 900 python -m pytest -x -q tests/test_gpu_tc.py tests/test_gpu_network.py tests/test_gpu_benchconfig.py 2>&1 | tail -2
bash scripts/ab_libs.sh "timeout 300 python scripts/frame_probe.py --profile | tail -3 | head -1 | grep -o 'conv_tc_tail.4.=[0-9.]*us'" base.so defer.so
bash scripts/ab_libs.sh "timeout 300 python bench.py --quick --steps 30 --streams 16 2>/dev/null | tail -1 | cut -c1-90" base.so defer.so
