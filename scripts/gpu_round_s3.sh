mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1; nproc > gpurun_out/nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_s3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_s3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s3.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_s3.log
for c in c4 c1 c2 c3 c5; do timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_s3.json 2> gpurun_out/bench_${c}_s3.err; done
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_s3.json 2> gpurun_out/bench_ref_s3.err
