# Round-2 GPU pass: gpu tests, default bench (C5), C2/C4 bench lines, reference arm.
# usage: bash tools/gpu_r02.sh TAG [configs...]
TAG=${1:-r}; shift
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -32 gpurun_out/pytest_gpu_$TAG.log
python bench.py > gpurun_out/bench_$TAG.log 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -1 gpurun_out/bench_$TAG.log | cut -c1-3000
tail -5 gpurun_out/bench_$TAG.err
for c in "$@"; do
  python bench.py --config $c --no-cpu > gpurun_out/bench_${c}_$TAG.log 2>&1; echo "bench $c rc=$?"
  tail -1 gpurun_out/bench_${c}_$TAG.log | cut -c1-1500
done
