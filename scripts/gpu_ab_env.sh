# A/B of one environment switch on the same library: $1 = "VAR=value" for the B arm; $2 = pytest filter
mkdir -p gpurun_out
if [ -n "$2" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$2" > gpurun_out/ab_pytest.log 2>&1; echo rc=$? >> gpurun_out/ab_pytest.log; fi
for i in 1 2 3; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e ${BENCH_ARGS:-} > gpurun_out/ab_new_$i.json 2>/dev/null
  env $1 timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e ${BENCH_ARGS:-} > gpurun_out/ab_old_$i.json 2>/dev/null
done
