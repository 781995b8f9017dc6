#!/bin/bash
# ncu --set full of the sketch kernels (one launch each) at the given shape (default c4).
tag=${1:-r01}; shift
shape=${@:-2048 1048576 0 1}
mkdir -p gpurun_out
for k in hchain_kernel fft_pass_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 2 \
    -o gpurun_out/sketch_${k}_$tag -f python scripts/bench_sketch.py $shape > gpurun_out/ncu_sketch_${k}_$tag.log 2>&1
done
