#!/bin/bash
# Round 2: CSNE-to-floor check, acceptance + full-size parity tests, parity campaign refresh
mkdir -p gpurun_out
timeout 600 python scripts/exp/accuracy_variants.py c2 > gpurun_out/acc_c2_c.log 2>&1
timeout 900 python scripts/exp/accuracy_variants.py c5s > gpurun_out/acc_c5s_c.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu_r02c.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r02c.log
timeout 3000 python scripts/parity_full.py --configs c1,c2,c3,c5s,c4,c5a --out gpurun_out/parity_c.json > gpurun_out/parity_c.log 2>&1
echo "parity rc=$?" >> gpurun_out/parity_c.log
