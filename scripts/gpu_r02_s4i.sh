#!/bin/bash
# session-4 final pass: GPU suite, smoke, same-box A/B of every config against the library QR path,
# the default bench line (c4 with e2e and the CPU baseline), device traces
mkdir -p gpurun_out/s4i
O=gpurun_out/s4i
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in c1 c2 c3 c4 c5; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
  MNB_QR_LIB=1 MNB_CHAIN_MIN_CHUNKS=16 timeout 600 python bench.py --config $c --no-cpu --no-e2e > $O/bench_${c}_lib.json 2> $O/bench_${c}_lib.err
  MNB_TRACE=1 timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 1 --warmup 2 > $O/trace_$c.json 2> $O/trace_$c.err
done
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
