#!/bin/bash
# Same-box A/B: staged draw with theta / d / sample held back (default) vs all draws at once (MNB_STAGED_DEFER=0);
# then the full-size parity campaign at the final code.
tag=${1:-ab6}
O=gpurun_out/$tag
mkdir -p $O
run() {  # name config env...
  local name=$1 c=$2; shift 2
  env "$@" timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 8 --warmup 3 > $O/bench_${c}_$name.json 2> $O/bench_${c}_$name.err
  env "$@" MNB_TRACE=1 timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 1 --warmup 2 > /dev/null 2> $O/trace_${c}_$name.err
  grep "device:\|staged\|build_srft" $O/trace_${c}_$name.err | tail -4 > $O/trace_${c}_$name.txt; rm -f $O/trace_${c}_$name.err
}
for rep in a b c; do
  run defer_$rep c4 MNB_X=0
  run nodefer_$rep c4 MNB_STAGED_DEFER=0
done
for rep in a b; do
  run defer_$rep c3 MNB_X=0
  run nodefer_$rep c3 MNB_STAGED_DEFER=0
  run defer_$rep c5 MNB_X=0
  run nodefer_$rep c5 MNB_STAGED_DEFER=0
done
O=$O python - <<'P' > $O/summary.txt
import json, glob, os
for f in sorted(glob.glob(os.environ['O'] + '/bench_*.json')):
    try:
        d = json.load(open(f)); print(os.path.basename(f), round(1e3 * d['value'], 3), 'ms median', round(d['ms_per_step_median'], 3), d['solve']['lsq_iterations'])
    except Exception as e:
        print(os.path.basename(f), 'ERR', e)
P
cat $O/summary.txt
grep -h "staged" $O/trace_c4_*.txt $O/trace_c5_*.txt
