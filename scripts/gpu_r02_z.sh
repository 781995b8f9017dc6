#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --config c5 --steps 1 --warmup 0 --no-e2e --no-cpu"
timeout 900 $CMD > gpurun_out/plain_c5z.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"fft_select_blocked8" -s 0 -c 1 \
  -o gpurun_out/fb8_c5 -f $CMD > gpurun_out/ncu_fb8.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_fb8.log
