#!/bin/bash
# round-end evidence at the final code: the c4 profile pass (launch list + ncu summaries) and the full-size parity campaign
bash scripts/profile_round.sh r02b > gpurun_out/profile_round_r02b.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
for k in chol_upper_kernel trtri_upper_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o /tmp/${k}_c4 -f $B > gpurun_out/prof_r02b/ncu_${k}.log 2>&1
  python scripts/ncu_summary.py /tmp/${k}_c4.ncu-rep > gpurun_out/prof_r02b/ncu_${k}_summary.txt 2>&1
done
timeout 2400 python scripts/parity_full.py --out gpurun_out/parity_s4j.json > gpurun_out/parity_full_s4j.log 2>&1
ls gpurun_out/prof_r02b
