# A/B: the built library vs gpurun_base/ (MNB_LIB_PATH), alternating runs; optional pytest filter $1
mkdir -p gpurun_out
if [ -n "$1" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/ab_pytest.log 2>&1; echo rc=$? >> gpurun_out/ab_pytest.log; fi
for i in 1 2 3; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e ${BENCH_ARGS:-} > gpurun_out/ab_new_$i.json 2>/dev/null
  MNB_LIB_PATH=$PWD/gpurun_base/libminnorm_b200.so timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e ${BENCH_ARGS:-} > gpurun_out/ab_old_$i.json 2>/dev/null
done
