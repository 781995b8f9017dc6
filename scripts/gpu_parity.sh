#!/bin/bash
# Full-size parity campaign on one B200 (scripts/parity_full.py); output merged back under gpurun_out/.
mkdir -p gpurun_out
cfgs=${1:-c1,c2,c3,c5a,c4}
timeout 3000 python scripts/parity_full.py --configs $cfgs --out gpurun_out/parity.json > gpurun_out/parity.log 2>&1
echo "rc=$?" >> gpurun_out/parity.log
