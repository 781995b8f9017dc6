#!/bin/bash
# A/B the fused pass across alternative builds of the library on one box:
#   bash scripts/ab_pass.sh "<m n real ...>" ab/lib_x.so ab/lib_y.so ...
# Each variant runs in its own process (MNB_LIB_PATH), twice, interleaved.
shapes=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib rep $rep"
    MNB_LIB_PATH=$PWD/$lib timeout 300 python scripts/bench_pass.py $shapes 2>&1 | grep '"ms"'
  done
done
