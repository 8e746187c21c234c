# sweep K1 tiles: bash tools/gpu_tune_k1.sh CONFIG "i j k"
CFG=$1; IDX=$2
for i in default $IDX; do
  if [ "$i" = default ]; then unset POLY_K1_TUNE; else export POLY_K1_TUNE=$i; fi
  timeout 600 python bench.py --config $CFG --steps ${STEPS:-100} --no-cpu --no-e2e > gpurun_out/tune_${CFG}_$i.log 2>&1
  tail -1 gpurun_out/tune_${CFG}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$CFG', '$i', d['config']['tile'], 'kernel_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],3), 'clk', d['clocks']['sm_mhz'] if d['clocks'] else None)" 2>&1 | tail -1
done
