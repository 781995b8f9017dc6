# bench lines for every BASELINE config + the reference arm + classical comparisons (no ncu)
mkdir -p gpurun_out
tag=${1:-final}
for c in c4 c1 c2 c3 c5; do timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_$tag.json 2> gpurun_out/bench_${c}_$tag.err; done
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
for c in c2 c3 c4 c5; do timeout 1200 python bench.py --config $c --steps 2 --warmup 2 --no-cpu --no-e2e --classical > gpurun_out/classical_${c}_$tag.json 2> gpurun_out/classical_${c}_$tag.err; done
