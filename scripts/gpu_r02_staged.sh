#!/bin/bash
# Same-box A/B of the staged draw of T (MNB_STAGED_DRAW=0: the one-shot draw + upload), then the GPU suite.
# usage: bash scripts/gpu_r02_staged.sh [tag]
tag=${1:-staged}
O=gpurun_out/$tag
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
for c in c4 c3 c5 c2; do
  for v in on off; do
    if [ $v = off ]; then export MNB_STAGED_DRAW=0; else unset MNB_STAGED_DRAW; fi
    timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 > $O/bench_${c}_$v.json 2> $O/bench_${c}_$v.err
    MNB_TRACE=1 timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 1 --warmup 2 > /dev/null 2> $O/trace_${c}_$v.err
    grep "device\|staged\|build_srft" $O/trace_${c}_$v.err | tail -6 > $O/trace_${c}_$v.txt; rm -f $O/trace_${c}_$v.err
  done
done
unset MNB_STAGED_DRAW
MNB_STAGED_MIN_N=1024 timeout 600 python bench.py --config c2 --no-cpu --no-e2e --steps 5 --warmup 3 > $O/bench_c2_min1024.json 2> $O/bench_c2_min1024.err
MNB_STAGED_MIN_N=1024 timeout 600 python bench.py --config c1 --no-cpu --no-e2e --steps 5 --warmup 3 > $O/bench_c1_min1024.json 2> $O/bench_c1_min1024.err
timeout 600 python bench.py --config c1 --no-cpu --no-e2e --steps 5 --warmup 3 > $O/bench_c1_on.json 2> $O/bench_c1_on.err
O=$O python - <<'P' > $O/summary.txt
import json, glob, os
for f in sorted(glob.glob(os.environ.get('O', 'gpurun_out/staged') + '/bench_*.json')):
    try:
        d = json.load(open(f)); print(os.path.basename(f), round(1e3 * d['value'], 3), 'ms', d['ms_per_step_all'], d['solve']['lsq_iterations'])
    except Exception as e:
        print(os.path.basename(f), 'ERR', e)
P
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
cat $O/summary.txt
