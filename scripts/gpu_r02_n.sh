#!/bin/bash
# Round 2: pass B half tiles (c4) -- sketch parity at n = 2^20, A/B bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x > gpurun_out/pytest_n.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_n.log
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4_half.json 2> gpurun_out/bench_c4_half.err
MNB_FB_HALF=0 timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4_full.json 2> gpurun_out/bench_c4_full.err
