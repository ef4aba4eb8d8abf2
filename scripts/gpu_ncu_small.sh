# usage: bash scripts/gpu_ncu_small.sh TAG "regex1 regex2 ..." -- ncu --set full of one steady launch of each kernel
TAG=${1:-small}; KS=${2:-"conv_planar detect_bits_kernel dilate_compact_kernel point_work_kernel point_scan_kernel conv_tc_kernel<1"}
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
for K in $KS; do
  N=$(echo "$K" | tr -cd 'a-z_')
  timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$K" --launch-skip 4 -c 1 \
    -o gpurun_out/${TAG}_${N} $B > gpurun_out/${TAG}_${N}.out 2>&1
  echo "$K rc=$?"
done
