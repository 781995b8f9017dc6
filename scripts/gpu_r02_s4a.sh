#!/bin/bash
# session-4 first pass: GPU suite at HEAD, smoke, default bench, traced small-config solves
mkdir -p gpurun_out/s4a
O=gpurun_out/s4a
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in c1 c2 c3; do
  timeout 300 python bench.py --config $c --no-cpu --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
  MNB_TRACE=1 timeout 300 python bench.py --config $c --no-cpu --no-e2e --steps 2 --warmup 3 > $O/trace_$c.json 2> $O/trace_$c.err
done
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
MNB_TRACE=1 timeout 300 python bench.py --config c4 --no-cpu --no-e2e --steps 2 --warmup 3 > $O/trace_c4.json 2> $O/trace_c4.err
ls -la $O
