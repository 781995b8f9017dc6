mkdir -p gpurun_out
MNB_TRACE=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/trace_c4.json 2> gpurun_out/trace_c4.err
MNB_TRACE=1 timeout 600 python bench.py --config c5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/trace_c5.json 2> gpurun_out/trace_c5.err
bash scripts/profile_round.sh s3
