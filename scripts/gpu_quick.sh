# quick GPU iteration: parity tests (optionally filtered) + one traced c4 bench
mkdir -p gpurun_out
tag=${1:-q}; filt=${2:-}
timeout 900 python -m pytest tests -m gpu -x -q ${filt:+-k "$filt"} > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
for c in ${CONFIGS:-c4}; do
MNB_TRACE=1 timeout 600 python bench.py --config $c --steps 3 --warmup 3 ${BENCH_ARGS:---no-cpu} > gpurun_out/bench_${c}_$tag.json 2> gpurun_out/bench_${c}_$tag.err
done
