#!/bin/bash
# Round 2: incremental Gram of E (c5, c4 host-A path) A/B + tests
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_dist.py tests/test_gpu_parity_full.py -q -x -k "not c4 and not c3" > gpurun_out/pytest_v.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v.log
MNB_TRACE=1 timeout 900 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_c5_v.json 2> gpurun_out/bench_c5_v.err
MNB_GRAM_AFTER=1 timeout 900 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_c5_v0.json 2> gpurun_out/bench_c5_v0.err
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c4_v.json 2> gpurun_out/bench_c4_v.err
MNB_GRAM_AFTER=1 timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c4_v0.json 2> gpurun_out/bench_c4_v0.err
