#!/bin/bash
# Same-box A/B of the host-A (e2e) path: S's Gram built slab by slab during the copy (default) vs after it
# (MNB_GRAM_S_AFTER=1); device timelines; then the GPU suite.
tag=${1:-ab11}
O=gpurun_out/$tag
mkdir -p $O
run() {  # name env...
  local name=$1; shift
  env "$@" timeout 900 python bench.py --no-cpu --steps 4 --warmup 3 > $O/bench_c4_$name.json 2> $O/bench_c4_$name.err
}
for rep in a b c; do
  run new_$rep MNB_X=0
  run after_$rep MNB_GRAM_S_AFTER=1
done
MNB_TRACE=1 timeout 900 python bench.py --no-cpu --steps 1 --warmup 2 > /dev/null 2> $O/trace_new.err
MNB_GRAM_S_AFTER=1 MNB_TRACE=1 timeout 900 python bench.py --no-cpu --steps 1 --warmup 2 > /dev/null 2> $O/trace_after.err
for v in new after; do grep "H2D done\|slab 7\|device cholqr" $O/trace_$v.err | tail -5 > $O/trace_$v.txt; rm -f $O/trace_$v.err; done
O=$O python - <<'P' > $O/summary.txt
import json, glob, os
for f in sorted(glob.glob(os.environ['O'] + '/bench_*.json')):
    try:
        d = json.load(open(f)); print(os.path.basename(f), 'value', round(1e3 * d['value'], 2), 'ms  e2e', round(1e3 * d['e2e']['value'], 2), 'ms')
    except Exception as e:
        print(os.path.basename(f), 'ERR', e)
P
cat $O/summary.txt; cat $O/trace_new.txt; echo ===; cat $O/trace_after.txt
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
