#!/bin/bash
# Round 2: c5 pass B with 2-row units (2 CTAs / SM) vs 4-row units; parity tests at n = 3*2^20
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -k "3145728 or multislab or c5 or real" > gpurun_out/pytest_j.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_j.log
timeout 900 python bench.py --config c5 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_c5_fb2.json 2> gpurun_out/bench_c5_fb2.err
MNB_FB_ROWS=4 timeout 900 python bench.py --config c5 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_c5_fb4.json 2> gpurun_out/bench_c5_fb4.err
