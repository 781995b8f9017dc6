mkdir -p gpurun_out
tag=${1:-fb}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sketch or fused" > gpurun_out/pytest_$tag.log 2>&1; echo rc=$? >> gpurun_out/pytest_$tag.log
MNB_TRACE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4_$tag.json 2> gpurun_out/bench_c4_$tag.err
K=${KERNEL:-fft1024_select_kernel}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o /tmp/k_$tag -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_$tag.log 2>&1
python scripts/ncu_summary.py /tmp/k_$tag.ncu-rep > gpurun_out/ncu_${tag}_summary.txt 2>&1
ncu -i /tmp/k_$tag.ncu-rep --page source --csv > gpurun_out/ncu_${tag}_source.csv 2>/dev/null
