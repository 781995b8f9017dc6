#!/bin/bash
# Round 2: early hand-over to shifted CholeskyQR3 (c3), QR tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -x > gpurun_out/pytest_o.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_o.log
for c in c2 c3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_${c}_o.json 2> gpurun_out/bench_${c}_o.err
done
MNB_TRACE=1 timeout 300 python bench.py --config c3 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2> gpurun_out/trace_c3_o.err
timeout 900 python -m pytest tests/test_gpu_parity_full.py -q -x -k "c3 or c2" > gpurun_out/pytest_o_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_o_full.log
