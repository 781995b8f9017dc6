#!/bin/bash
# the fused H + pass A path at n1 = 128 ... 512 (c3) with the direct pruned pass B
mkdir -p gpurun_out/s4l
O=gpurun_out/s4l
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_api.py -x -q > $O/pytest_part.log 2>&1; echo "rc=$?" >> $O/pytest_part.log
for c in c3 c2; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
  MNB_FFT_BALANCED=1 timeout 600 python bench.py --config $c --no-cpu --no-e2e > $O/bench_${c}_balanced.json 2> $O/bench_${c}_balanced.err
done
MNB_TRACE=1 timeout 600 python bench.py --config c3 --no-cpu --no-e2e --steps 1 --warmup 2 > $O/trace_c3.json 2> $O/trace_c3.err
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
MNB_NO_VERDICT=1 timeout 600 python bench.py --config c3 --no-cpu --no-e2e > $O/bench_c3_noverdict.json 2> $O/bench_c3_noverdict.err
timeout 600 python bench.py --config c1 --no-cpu --no-e2e > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c4 --no-cpu --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err
