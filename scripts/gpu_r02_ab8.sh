#!/bin/bash
# Same-box A/B, more repetitions: 16 vs 14 host threads for the parameter draw (MNB_HOST_THREADS).
tag=${1:-ab8}
O=gpurun_out/$tag
mkdir -p $O
run() {  # name config env...
  local name=$1 c=$2; shift 2
  env "$@" timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 10 --warmup 3 > $O/bench_${c}_$name.json 2> $O/bench_${c}_$name.err
}
for rep in a b c d; do
  run t16_$rep c4 MNB_X=0
  run t14_$rep c4 MNB_HOST_THREADS=14
done
for rep in a b c; do
  run t16_$rep c5 MNB_X=0
  run t14_$rep c5 MNB_HOST_THREADS=14
  run t16_$rep c3 MNB_X=0
  run t14_$rep c3 MNB_HOST_THREADS=14
done
O=$O python - <<'P' > $O/summary.txt
import json, glob, os
for f in sorted(glob.glob(os.environ['O'] + '/bench_*.json')):
    try:
        d = json.load(open(f)); print(os.path.basename(f), round(1e3 * d['value'], 3), 'ms median', round(d['ms_per_step_median'], 3), 'step0 host s', round(d['solve']['step_seconds'][0], 5), 'param', round(d['solve']['param_seconds'], 5))
    except Exception as e:
        print(os.path.basename(f), 'ERR', e)
P
cat $O/summary.txt
