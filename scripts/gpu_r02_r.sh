#!/bin/bash
# Round 2: merged CG update kernel A/B (c3, c4, c5) + tests
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_dist.py tests/test_gpu_parity_full.py -q -x > gpurun_out/pytest_r.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r.log
for c in c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_${c}_r.json 2> gpurun_out/bench_${c}_r.err
  MNB_CG_UPD3=1 timeout 900 python bench.py --config $c --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_${c}_r3.json 2> gpurun_out/bench_${c}_r3.err
done
