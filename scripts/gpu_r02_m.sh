#!/bin/bash
# Round 2: concurrent QR(E) (helper thread) -- GPU suite + per-config bench lines
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_m.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_m.log
for c in c1 c2 c3 c4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_${c}_m.json 2> gpurun_out/bench_${c}_m.err
done
MNB_TRACE=1 timeout 300 python bench.py --config c3 --steps 1 --warmup 2 --no-cpu --no-e2e > /dev/null 2> gpurun_out/trace_c3_m.err
