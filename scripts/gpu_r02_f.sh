#!/bin/bash
# Round 2: persistent small-problem CG (c1/c2 A/B), full GPU suite (reproduce the in-suite c4 failure)
mkdir -p gpurun_out
for c in c1 c2; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_${c}_small.json 2> gpurun_out/bench_${c}_small.err
  MNB_SMALL_CG_OFF=1 timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_${c}_multi.json 2> gpurun_out/bench_${c}_multi.err
done
timeout 1800 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/pytest_gpu_r02f.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r02f.log
