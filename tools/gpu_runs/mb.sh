set -u
mkdir -p gpurun_out/mb
timeout 120 tools/microbench/mma_shape > gpurun_out/mb/mma_shape.txt 2>&1
