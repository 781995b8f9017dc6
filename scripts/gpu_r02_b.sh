#!/bin/bash
# Round 2: distributed (world-1 NCCL) + multi-slab GPU tests, accuracy diagnostics at c2 / c5-like
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dist.log
timeout 600 python scripts/exp/accuracy_variants.py c2 > gpurun_out/acc_c2.log 2>&1
timeout 900 python scripts/exp/accuracy_variants.py c5s > gpurun_out/acc_c5s.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r02b.log
