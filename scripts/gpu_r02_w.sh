#!/bin/bash
mkdir -p gpurun_out
MNB_TRACE=1 timeout 300 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2> gpurun_out/trace_c2_w.err
MNB_TRACE=1 timeout 300 python bench.py --config c1 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2> gpurun_out/trace_c1_w.err
