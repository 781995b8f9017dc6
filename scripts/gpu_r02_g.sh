#!/bin/bash
# Round 2: c2 timeline trace, full GPU suite (reproduce the in-suite c4 failure)
mkdir -p gpurun_out
MNB_TRACE=1 timeout 300 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/trace_c2.json 2> gpurun_out/trace_c2.err
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu_r02g.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r02g.log
