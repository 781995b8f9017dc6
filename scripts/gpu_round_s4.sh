# Full refresh: GPU tests, smoke, c1..c5 + reference bench lines, c4 launch list + ncu summaries.
mkdir -p gpurun_out
tag=${1:-s4}
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$tag.log
for c in c4 c1 c2 c3 c5; do timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_$tag.json 2> gpurun_out/bench_${c}_$tag.err; done
for c in c2 c3 c4; do timeout 900 python bench.py --config $c --steps 2 --warmup 2 --no-cpu --no-e2e --classical > gpurun_out/classical_${c}_$tag.json 2> gpurun_out/classical_${c}_$tag.err; done
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
bash scripts/profile_round.sh $tag
