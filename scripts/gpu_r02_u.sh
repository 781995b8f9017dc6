#!/bin/bash
# Round 2: full GPU suite after the stream-ordering fix
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=12 > gpurun_out/pytest_u.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_u.log
