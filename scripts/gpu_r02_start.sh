#!/bin/bash
# Round-2 first GPU pass: box probe, GPU tests, smoke, default bench, then the full-size parity campaign.
mkdir -p gpurun_out
(nproc; free -g; lscpu | head -20; nvidia-smi) > gpurun_out/box_probe.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r02a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02a.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_r02a.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_c4_r02a.json 2> gpurun_out/bench_c4_r02a.err
timeout 3000 python scripts/parity_full.py --configs ${1:-c1,c2,c3,c5a,c4} --out gpurun_out/parity.json > gpurun_out/parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/parity.log
