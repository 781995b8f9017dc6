mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "solve or lsq or least or classical or init or csne" > gpurun_out/ab_pytest.log 2>&1; echo rc=$? >> gpurun_out/ab_pytest.log
for c in c2 c4; do for i in 1 2; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_new_${c}_$i.json 2>/dev/null
  MNB_LIB_PATH=$PWD/gpurun_base/libminnorm_b200.so timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_old_${c}_$i.json 2>/dev/null
done; done
