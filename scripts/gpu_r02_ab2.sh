#!/bin/bash
# Same-box A/B: early Cholesky verdict of QR(S) (c3), T' uploaded on the copy stream, helper stream priority.
# usage: bash scripts/gpu_r02_ab2.sh [tag]
tag=${1:-ab2}
O=gpurun_out/$tag
mkdir -p $O
run() {  # name config env...
  local name=$1 c=$2; shift 2
  env "$@" timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 5 --warmup 3 > $O/bench_${c}_$name.json 2> $O/bench_${c}_$name.err
  env "$@" MNB_TRACE=1 timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 1 --warmup 2 > /dev/null 2> $O/trace_${c}_$name.err
  grep "device\|staged\|fast QR\|chain" $O/trace_${c}_$name.err | tail -8 > $O/trace_${c}_$name.txt; rm -f $O/trace_${c}_$name.err
}
run default c3 MNB_X=0
run noearly c3 MNB_EARLY_VERDICT=0
run noside c3 MNB_SIDE_UPLOAD=0
run prio c3 MNB_QR_PRIO=1
run default2 c3 MNB_X=0
run default c4 MNB_X=0
run noside c4 MNB_SIDE_UPLOAD=0
run prio c4 MNB_QR_PRIO=1
run default c5 MNB_X=0
run noside c5 MNB_SIDE_UPLOAD=0
run default c2 MNB_X=0
run prio c2 MNB_QR_PRIO=1
run default c1 MNB_X=0
O=$O python - <<'P' > $O/summary.txt
import json, glob, os
for f in sorted(glob.glob(os.environ['O'] + '/bench_*.json')):
    try:
        d = json.load(open(f)); print(os.path.basename(f), round(1e3 * d['value'], 3), 'ms', [round(x, 2) for x in d['ms_per_step_all']], d['solve']['lsq_iterations'])
    except Exception as e:
        print(os.path.basename(f), 'ERR', e)
P
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
cat $O/summary.txt
