#!/bin/bash
# Round 2: small-CG + sync-free power steps (c1/c2/c3 bench), c4 stress, c5 full solve trace
mkdir -p gpurun_out
for c in c1 c2 c3; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_${c}_h.json 2> gpurun_out/bench_${c}_h.err
done
MNB_TRACE=1 timeout 300 python bench.py --config c2 --steps 2 --warmup 2 --no-cpu --no-e2e > /dev/null 2> gpurun_out/trace_c2_h.err
timeout 900 python scripts/exp/stress_c4.py c4 6 > gpurun_out/stress_c4.log 2>&1
MNB_TRACE=1 timeout 900 python bench.py --config c5 --steps 2 --warmup 1 --no-cpu --no-e2e --classical > gpurun_out/bench_c5_h.json 2> gpurun_out/bench_c5_h.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_dist.py -q -x > gpurun_out/pytest_h.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_h.log
