# detect with 64 registers (two CTAs beside the other lane's layer 3) vs 74-78
bash scripts/ab_libs.sh "timeout 300 python bench.py --quick --steps 30 --streams 16 2>/dev/null | tail -1 | cut -c1-90" base.so det4.so
cp paper_1704_04313_b200/_lib_alt/det4.so paper_1704_04313_b200/_lib/libcbx.so
timeout 300 python scripts/timeline_probe.py --steps 2 2>&1 | grep -E "detect|dilate_compact_kernel<4|span"
