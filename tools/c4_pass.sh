# C4 pass timing: ring kernels vs the plain SELL16 kernels, plus parity tests.
mkdir -p gpurun_out
TAG=${1:-c4}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "c4 or dsell" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
for v in dsell sell16; do
  if [ $v = sell16 ]; then export POLY_NO_DSELL=1; else unset POLY_NO_DSELL; fi
  python bench.py --config c4 --no-cpu --no-e2e --steps 200 > gpurun_out/bench_c4_${v}_$TAG.log 2>&1; echo "bench $v rc=$?"
  python - <<PY
import json
l=json.loads(open("gpurun_out/bench_c4_${v}_$TAG.log").read().strip().splitlines()[-1])
r=l["roofline"]
print("$v", "step_ms", round(l["ms_per_step"]*1e3,1), "pass_us", round(r["kernel_ms"]*1e3,1), "fin_us", round(r["finalize_ms"]*1e3,1), "frac", round(r["frac"],3))
PY
done
unset POLY_NO_DSELL
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_dsell|k_sell16" -s 8 -c 4 python bench.py --config c4 --no-cpu --no-e2e --steps 4 --warmup 3 > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
grep -E "k_dsell|k_sell16|duration|dram__bytes|warps_active|l1tex__thr|lts__thr" gpurun_out/ncu_$TAG.log | head -40
