#!/bin/bash
# Round 2: GEMV power steps (c5 QR(E)), e2e timeline at c4, QR tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -x > gpurun_out/pytest_q.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q.log
MNB_TRACE=1 timeout 900 python bench.py --config c5 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_c5_q.json 2> gpurun_out/bench_c5_q.err
MNB_TRACE=1 timeout 900 python bench.py --config c4 --steps 2 --warmup 2 --no-cpu > gpurun_out/bench_c4_q.json 2> gpurun_out/bench_c4_q.err
