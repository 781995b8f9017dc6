mkdir -p gpurun_out
for v in 1 2 4 8 16 64; do
  MNB_P2FA_SYNC=$v timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_c4_sync$v.json 2> gpurun_out/bench_c4_sync$v.err
done
