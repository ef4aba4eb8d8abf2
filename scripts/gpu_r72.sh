# ncu of the L2 conv (steady frame): production build and the timing-only build without gather/stores/B refetch
mkdir -p gpurun_out
for L in base l2all; do
cp paper_1704_04313_b200/_lib_alt/$L.so paper_1704_04313_b200/_lib/libcbx.so
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:conv_tc_kernel<.bool.1, .int.0, .bool.0" -s 3 -c 1 \
  -o gpurun_out/r72_$L python scripts/frame_probe.py --frames 6 > gpurun_out/r72_$L.out 2>&1; echo "$L rc=$?"
done
