mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/mma_shape_probe scripts/mma_shape_probe.cu && timeout 300 ./gpurun_out/mma_shape_probe 2>&1 | tee gpurun_out/r2o_mma_shape.log
rm -f gpurun_out/mma_shape_probe
