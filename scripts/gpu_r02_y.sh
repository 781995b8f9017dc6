#!/bin/bash
# Round 2: radix-8 two-row pass B at N = 3072 (c5) -- parity tests at n = 3*2^20, A/B bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -k "3145728 or multislab or real" > gpurun_out/pytest_y.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_y.log
timeout 900 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_c5_r8.json 2> gpurun_out/bench_c5_r8.err
MNB_FB_RADIX=16 timeout 900 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_c5_r16.json 2> gpurun_out/bench_c5_r16.err
