#!/bin/bash
# Same-box A/B of a kernel change: the library built before it (libminnorm_b200_prev.so, MNB_LIB_PATH)
# against the current one, on the sketch-heavy configs; then the fused-pass parity tests.
tag=${1:-ab5}
O=gpurun_out/$tag
mkdir -p $O
PREV=$PWD/paper_0905_4745_b200/libminnorm_b200_prev.so
run() {  # name config env...
  local name=$1 c=$2; shift 2
  env "$@" timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 8 --warmup 3 > $O/bench_${c}_$name.json 2> $O/bench_${c}_$name.err
}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_parity.log 2>&1; echo "pytest rc=$?" >> $O/pytest_parity.log
tail -3 $O/pytest_parity.log
for rep in a b; do
  run new_$rep c4 MNB_X=0
  run prev_$rep c4 MNB_LIB_PATH=$PREV
  run new_$rep c3 MNB_X=0
  run prev_$rep c3 MNB_LIB_PATH=$PREV
done
run new c5 MNB_X=0
run prev c5 MNB_LIB_PATH=$PREV
O=$O python - <<'P' > $O/summary.txt
import json, glob, os
for f in sorted(glob.glob(os.environ['O'] + '/bench_*.json')):
    try:
        d = json.load(open(f)); print(os.path.basename(f), round(1e3 * d['value'], 3), 'ms median', round(d['ms_per_step_median'], 3), d['solve']['lsq_iterations'], {k: round(v, 2) for k, v in d['solve']['sketch_kernel_ms'].items()})
    except Exception as e:
        print(os.path.basename(f), 'ERR', e)
P
cat $O/summary.txt
