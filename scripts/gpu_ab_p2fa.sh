# A/B of the fused pass: the built library vs the committed one (MNB_LIB_PATH), alternating runs
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ab_new_$i.json 2>/dev/null
  MNB_LIB_PATH=$PWD/gpurun_base/libminnorm_b200.so timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ab_old_$i.json 2>/dev/null
done
