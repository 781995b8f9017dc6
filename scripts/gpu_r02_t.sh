#!/bin/bash
# Round 2: full GPU suite with MNB_TRACE (captured per failing test) to catch the intermittent
# non-converged first solve at c4/c5 inside the suite
mkdir -p gpurun_out
MNB_TRACE=1 timeout 2400 python -m pytest tests -m gpu -q -x -p no:randomly > gpurun_out/pytest_t.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_t.log
