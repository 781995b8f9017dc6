#!/bin/bash
# same-box A/B: ab/lib_prev.so (A) vs the tree's library (B), alternating
mkdir -p gpurun_out
CFG=${1:-c5}
for i in 1 2; do
  MNB_LIB_PATH=$PWD/ab/lib_prev.so timeout 900 python bench.py --config $CFG --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/ab_A$i.json 2> gpurun_out/ab_A$i.err
  timeout 900 python bench.py --config $CFG --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/ab_B$i.json 2> gpurun_out/ab_B$i.err
done
