# K4t iteration: K4t tests, C4 parity tests, C4 bench line.  usage: bash tools/gpu_k4.sh [pytest -k expr]
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_k4t.py -x -q > gpurun_out/k4t_tests.log 2>&1; echo "k4t tests rc=$?"; tail -3 gpurun_out/k4t_tests.log
timeout 900 python -m pytest tests -m gpu -x -q -k "${1:-c4 or C4 or csr or tiled}" > gpurun_out/c4_tests.log 2>&1; echo "c4 tests rc=$?"; tail -3 gpurun_out/c4_tests.log
timeout 300 python bench.py --config c4 --steps 100 --no-cpu --no-e2e > gpurun_out/bench_c4.log 2>&1; echo "c4 bench rc=$?"
python - <<'P'
import json
l = json.loads(open('gpurun_out/bench_c4.log').read().strip().splitlines()[-1])
r = l['roofline']
print('step_ms', l['ms_per_step'], 'pass_ms', r['kernel_ms'], 'frac', r['frac'])
P
