#!/bin/bash
# Round 2: first-solve diagnostic at c4 (fresh context), CLI GPU tests
mkdir -p gpurun_out
MNB_TRACE=1 timeout 900 python scripts/exp/first_solve.py c4 > gpurun_out/first_c4.log 2> gpurun_out/first_c4.err
timeout 600 python -m pytest tests/test_cli.py -x -q > gpurun_out/pytest_cli.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cli.log
