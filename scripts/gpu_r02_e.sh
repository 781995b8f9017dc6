#!/bin/bash
# Round 2: reproduce the in-pytest c4 non-convergence (full-size parity file alone, then after the suite)
mkdir -p gpurun_out
MNB_TRACE=1 timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -s > gpurun_out/pf_alone.log 2>&1; echo "rc=$?" >> gpurun_out/pf_alone.log
