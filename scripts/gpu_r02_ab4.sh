#!/bin/bash
# Same-box A/B: staged draw with / without deferring the other half's draws (MNB_STAGED_DEFER=0), then the GPU suite.
tag=${1:-ab4}
O=gpurun_out/$tag
mkdir -p $O
run() {  # name config env...
  local name=$1 c=$2; shift 2
  env "$@" timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 8 --warmup 3 > $O/bench_${c}_$name.json 2> $O/bench_${c}_$name.err
  env "$@" MNB_TRACE=1 timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 1 --warmup 2 > /dev/null 2> $O/trace_${c}_$name.err
  grep "device\|staged\|build_srft" $O/trace_${c}_$name.err | tail -4 > $O/trace_${c}_$name.txt; rm -f $O/trace_${c}_$name.err
}
for rep in a b; do
  run defer_$rep c4 MNB_X=0
  run nodefer_$rep c4 MNB_STAGED_DEFER=0
  run defer_$rep c3 MNB_X=0
  run nodefer_$rep c3 MNB_STAGED_DEFER=0
done
run defer c5 MNB_X=0
run nodefer c5 MNB_STAGED_DEFER=0
O=$O python - <<'P' > $O/summary.txt
import json, glob, os
for f in sorted(glob.glob(os.environ['O'] + '/bench_*.json')):
    try:
        d = json.load(open(f)); print(os.path.basename(f), round(1e3 * d['value'], 3), 'ms median', round(d['ms_per_step_median'], 3), d['solve']['lsq_iterations'])
    except Exception as e:
        print(os.path.basename(f), 'ERR', e)
P
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
cat $O/summary.txt
