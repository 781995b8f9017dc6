#!/bin/bash
# ncu --set full of one fused PCG pass launch at the given shape (default c4).
tag=${1:-r01}; shift
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcg_pass_kernel -s 3 -c 1 \
  -o gpurun_out/pcg_pass_$tag -f python scripts/bench_pass.py ${@:-2048 1048576 0} > gpurun_out/ncu_pass_$tag.log 2>&1
