#!/bin/bash
mkdir -p gpurun_out/s4d
O=gpurun_out/s4d
timeout 900 python -m pytest tests/test_gpu_cholqr.py -q > $O/pytest_cholqr.log 2>&1; echo "rc=$?" >> $O/pytest_cholqr.log
for c in c1 c2 c3 c4; do
  MNB_TRACE=1 timeout 300 python bench.py --config $c --no-cpu --no-e2e --steps 2 --warmup 3 > $O/trace_$c.json 2> $O/trace_$c.err
done
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for c in c1 c2 c3 c4 c5; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
done
