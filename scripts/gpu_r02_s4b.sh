#!/bin/bash
# session-4: the hand-written sketch-QR kernels -- unit tests, then the suite, then traced solves
mkdir -p gpurun_out/s4b
O=gpurun_out/s4b
timeout 900 python -m pytest tests/test_gpu_cholqr.py -x -q > $O/pytest_cholqr.log 2>&1; echo "rc=$?" >> $O/pytest_cholqr.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in c1 c2 c3 c4; do
  MNB_TRACE=1 timeout 300 python bench.py --config $c --no-cpu --no-e2e --steps 2 --warmup 3 > $O/trace_$c.json 2> $O/trace_$c.err
  timeout 300 python bench.py --config $c --no-cpu --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
