#!/bin/bash
# Round-end pass on one box: GPU suite, smoke, bench line of every config, the default bench line
# (c4 with e2e and the CPU baseline), the reference arm, launch list + ncu summaries of a c3 solve.
# usage: bash scripts/gpu_round_end.sh [tag]
tag=${1:-end}
O=gpurun_out/$tag
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in c1 c2 c3 c4 c5; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
  MNB_TRACE=1 timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 1 --warmup 2 > /dev/null 2> $O/trace_$c.err
  grep "device\|chain\|fast QR\|one-pass\|build_srft" $O/trace_$c.err | tail -10 > $O/trace_$c.txt; rm -f $O/trace_$c.err
done
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_reference.json 2> $O/bench_reference.err
B="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 900 ncu --nvtx --nvtx-include "solve/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c3.csv $B > $O/ncu_launch_c3.log 2>&1
python scripts/launch_summary.py $O/launches_c3.csv > $O/launches_c3_summary.txt 2>&1
for k in fft_select_blocked_direct_kernel p2fa_kernel sketch_refine_kernel; do
  timeout 900 ncu --nvtx --nvtx-include "solve/" --set full --clock-control none --import-source on \
    -k regex:$k -c 1 -o /tmp/${k}_c3 -f $B > $O/ncu_${k}.log 2>&1
  python scripts/ncu_summary.py /tmp/${k}_c3.ncu-rep > $O/ncu_${k}_c3_summary.txt 2>&1
done
ls -la $O
