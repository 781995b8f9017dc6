#!/bin/bash
# Same-box A/B: host threads of the parameter draw (MNB_HOST_THREADS; default = all 16 vCPUs).
tag=${1:-ab7}
O=gpurun_out/$tag
mkdir -p $O
run() {  # name config env...
  local name=$1 c=$2; shift 2
  env "$@" timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 8 --warmup 3 > $O/bench_${c}_$name.json 2> $O/bench_${c}_$name.err
  env "$@" MNB_TRACE=1 timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 1 --warmup 2 > /dev/null 2> $O/trace_${c}_$name.err
  grep "device:\|staged\|build_srft" $O/trace_${c}_$name.err | tail -4 > $O/trace_${c}_$name.txt; rm -f $O/trace_${c}_$name.err
}
for rep in a b; do
  run t16_$rep c4 MNB_X=0
  run t15_$rep c4 MNB_HOST_THREADS=15
  run t14_$rep c4 MNB_HOST_THREADS=14
  run t12_$rep c4 MNB_HOST_THREADS=12
done
run t16 c5 MNB_X=0
run t14 c5 MNB_HOST_THREADS=14
run t16 c3 MNB_X=0
run t14 c3 MNB_HOST_THREADS=14
O=$O python - <<'P' > $O/summary.txt
import json, glob, os
for f in sorted(glob.glob(os.environ['O'] + '/bench_*.json')):
    try:
        d = json.load(open(f)); print(os.path.basename(f), round(1e3 * d['value'], 3), 'ms median', round(d['ms_per_step_median'], 3), d['solve']['lsq_iterations'])
    except Exception as e:
        print(os.path.basename(f), 'ERR', e)
P
cat $O/summary.txt
grep -h "threads=1[0-9]\|staged" $O/trace_c4_*.txt | cut -c1-260
