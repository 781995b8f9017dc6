#!/bin/bash
# One gpurun pass: GPU parity tests, smoke, bench (c4 default + c2), ncu launch list,
# and one `ncu --set full` capture of the PCG pass and the H-stage kernel.
# usage (from the repo root on the box): bash scripts/gpu_check.sh [tag]
tag=${1:-r01}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1; nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$tag.log
timeout 900 python bench.py > gpurun_out/bench_c4_$tag.json 2> gpurun_out/bench_c4_$tag.err
timeout 300 python bench.py --config c2 > gpurun_out/bench_c2_$tag.json 2> gpurun_out/bench_c2_$tag.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_$tag.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcg_pass_kernel -s 2 -c 1 \
  -o gpurun_out/pcg_pass_c4_$tag -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_full_pcg_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hstage_kernel -s 0 -c 1 \
  -o gpurun_out/hstage_c4_$tag -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_full_hstage_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fft_pass_kernel -s 0 -c 1 \
  -o gpurun_out/fft_c4_$tag -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_full_fft_$tag.log 2>&1
fi
ls -la gpurun_out
