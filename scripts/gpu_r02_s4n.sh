#!/bin/bash
mkdir -p gpurun_out/s4n
O=gpurun_out/s4n
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for c in c1 c2 c3; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
  MNB_TRACE=1 timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 1 --warmup 2 > /dev/null 2> $O/trace_$c.err
  grep "device\|chain\|fast QR\|one-pass" $O/trace_$c.err | tail -8 > $O/trace_$c.txt
done
