#!/bin/bash
# Round 2: c5 fused-pass cluster-barrier interval sweep (MNB_P2FA_SYNC)
mkdir -p gpurun_out
for k in 16 4 64 1024; do
  MNB_P2FA_SYNC=$k timeout 600 python bench.py --config c5 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_c5_sync$k.json 2> gpurun_out/bench_c5_sync$k.err
done
