#!/bin/bash
# Round 2: c3 QR paths (shifted CholeskyQR3 vs Householder); CPU baseline (complete oracle solves) c1-c3
mkdir -p gpurun_out
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c3_default.json 2> gpurun_out/bench_c3_default.err
MNB_QR=householder timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c3_hh.json 2> gpurun_out/bench_c3_hh.err
MNB_TRACE=1 timeout 300 python bench.py --config c3 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2> gpurun_out/trace_c3.err
timeout 1500 python scripts/cpu_baseline.py --configs c1,c2,c3 --threads 1,all --out gpurun_out/cpu_baseline.json > gpurun_out/cpu_baseline.log 2>&1
