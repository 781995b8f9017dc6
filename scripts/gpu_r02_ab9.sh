#!/bin/bash
# Same-box A/B of the host-A (e2e) path: short last row slab + short slabs split into two k1 segments in the
# fused pass (default) vs eight equal slabs (MNB_EVEN_SLABS=1) vs the previous behaviour (+ MNB_P2FA_SEG=1).
tag=${1:-ab9}
O=gpurun_out/$tag
mkdir -p $O
run() {  # name env...
  local name=$1; shift
  env "$@" timeout 900 python bench.py --no-cpu --steps 4 --warmup 3 > $O/bench_c4_$name.json 2> $O/bench_c4_$name.err
}
for rep in a b; do
  run new_$rep MNB_X=0
  run even_$rep MNB_EVEN_SLABS=1
  run old_$rep MNB_EVEN_SLABS=1 MNB_P2FA_SEG=1
done
O=$O python - <<'P' > $O/summary.txt
import json, glob, os
for f in sorted(glob.glob(os.environ['O'] + '/bench_*.json')):
    try:
        d = json.load(open(f)); print(os.path.basename(f), 'value', round(1e3 * d['value'], 2), 'ms  e2e', round(1e3 * d['e2e']['value'], 2), 'ms')
    except Exception as e:
        print(os.path.basename(f), 'ERR', e)
P
cat $O/summary.txt
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
