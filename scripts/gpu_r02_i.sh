#!/bin/bash
# Round 2: classical TSQR tests; ncu --set full of the c5 sketch kernels (P1, fused P2+FA, pass B)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_dist.py tests/test_cli.py -q -x > gpurun_out/pytest_i.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_i.log
CMD="python bench.py --config c5 --steps 1 --warmup 0 --no-e2e --no-cpu"
timeout 900 $CMD > gpurun_out/plain_c5.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"hchain_kernel|p2fa_kernel|fft_select_blocked_kernel" -s 0 -c 3 \
  -o gpurun_out/sketch_c5_r02 -f $CMD > gpurun_out/ncu_c5.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_c5.log
