#!/bin/bash
mkdir -p gpurun_out/s4e
O=gpurun_out/s4e
timeout 600 python scripts/bench_cholqr.py > $O/bench_cholqr.log 2>&1; cp gpurun_out/bench_cholqr.json $O/ 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_cholqr.py tests/test_gpu_parity.py tests/test_gpu_api.py -x -q > $O/pytest_part.log 2>&1; echo "rc=$?" >> $O/pytest_part.log
for c in c1 c2; do
  MNB_TRACE=1 timeout 300 python bench.py --config $c --no-cpu --no-e2e --steps 2 --warmup 3 > $O/trace_$c.json 2> $O/trace_$c.err
  timeout 300 python bench.py --config $c --no-cpu --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
done
MNB_TINY_CG_OFF=1 timeout 300 python bench.py --config c1 --no-cpu --no-e2e > $O/bench_c1_tinyoff.json 2> $O/bench_c1_tinyoff.err
timeout 600 python bench.py --config c5 --no-cpu --no-e2e > $O/bench_c5_fast.json 2> $O/bench_c5_fast.err
MNB_FASTQR=0 timeout 600 python bench.py --config c5 --no-cpu --no-e2e > $O/bench_c5_fastoff.json 2> $O/bench_c5_fastoff.err
MNB_QR_LIB=1 timeout 600 python bench.py --config c5 --no-cpu --no-e2e > $O/bench_c5_lib.json 2> $O/bench_c5_lib.err
MNB_QR_LIB=1 timeout 600 python bench.py --config c4 --no-cpu --no-e2e > $O/bench_c4_lib.json 2> $O/bench_c4_lib.err
timeout 600 python bench.py --config c4 --no-cpu --no-e2e > $O/bench_c4_fast.json 2> $O/bench_c4_fast.err
MNB_QR_LIB=1 timeout 600 python bench.py --config c3 --no-cpu --no-e2e > $O/bench_c3_lib.json 2> $O/bench_c3_lib.err
timeout 600 python bench.py --config c3 --no-cpu --no-e2e > $O/bench_c3_fast.json 2> $O/bench_c3_fast.err
