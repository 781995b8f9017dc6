#!/bin/bash
# Round profile capture (run on the GPU box): launch list of one timed c4 solve
# (NVTX range "solve") and one `ncu --set full` capture per hot kernel, reduced
# on the box to text summaries (the full reports exceed gpurun's copy-back cap).
tag=${1:-r01}
mkdir -p gpurun_out/prof_$tag
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
# the same command line must have exited 0 without ncu first (B200_PROFILING.md)
timeout 900 $B > gpurun_out/prof_$tag/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --nvtx --nvtx-include "solve/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof_$tag/launches_c4.csv $B > gpurun_out/prof_$tag/ncu_launch.log 2>&1
python scripts/launch_summary.py gpurun_out/prof_$tag/launches_c4.csv > gpurun_out/prof_$tag/launches_c4_summary.txt 2>&1
for k in pcg_pass_kernel hchain_kernel p2fa_kernel fft1024_select_kernel p2fa_carry_kernel; do
  timeout 900 ncu --nvtx --nvtx-include "solve/" --set full --clock-control none --import-source on \
    -k regex:$k -c 2 -o /tmp/${k}_$tag -f $B > gpurun_out/prof_$tag/ncu_${k}.log 2>&1
  python scripts/ncu_summary.py /tmp/${k}_$tag.ncu-rep > gpurun_out/prof_$tag/ncu_${k}_summary.txt 2>&1
  ncu -i /tmp/${k}_$tag.ncu-rep --page details --csv > gpurun_out/prof_$tag/ncu_${k}_details.csv 2>/dev/null
done
cp /tmp/pcg_pass_kernel_$tag.ncu-rep gpurun_out/prof_$tag/ 2>/dev/null
du -sh gpurun_out/prof_$tag
