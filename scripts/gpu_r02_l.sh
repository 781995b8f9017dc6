#!/bin/bash
# Round 2: FP64 peaks, default bench (c4; complete CPU-port solve as cpu_baseline), reference arm,
# then the 1-thread c4 CPU baseline (long)
mkdir -p gpurun_out
timeout 300 python scripts/micro/fp64_peaks.py > gpurun_out/fp64_peaks.json 2> gpurun_out/fp64_peaks.err
mkdir -p profiles/r02 && cp gpurun_out/fp64_peaks.json profiles/r02/fp64_peaks.json
timeout 1200 python bench.py > gpurun_out/bench_c4_default.json 2> gpurun_out/bench_c4_default.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_c4.json 2> gpurun_out/bench_ref_c4.err
timeout 2700 python scripts/cpu_baseline.py --configs c4 --threads all,1 --out gpurun_out/cpu_baseline_c4.json > gpurun_out/cpu_baseline_c4.log 2>&1
