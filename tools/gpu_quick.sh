# quick GPU iteration: gpu tests (optional -k filter) + short bench lines
# usage: bash tools/gpu_quick.sh TAG "PYTEST_K" cfg1 cfg2 ...
TAG=$1; K=$2; shift 2
mkdir -p gpurun_out
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_$TAG.log
fi
for c in "$@"; do
  timeout 600 python bench.py --config $c --steps 100 --no-cpu --no-e2e > gpurun_out/bench_${c}_$TAG.log 2>&1; echo "bench $c rc=$?"
  tail -1 gpurun_out/bench_${c}_$TAG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['name'], 'value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],4), 'kernel_ms', round(r['kernel_ms'],4), 'fin_ms', round(r['finalize_ms'],4), 'frac', round(r['frac'],3))" 2>&1 | tail -2
done
