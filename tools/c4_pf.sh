# K4 software-pipelined stream loads (POLY_SELL_PF bits: 1 K4f, 2 K4b) A/B on C4
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c4_full or c4_solve" > /dev/null 2>&1; echo "pytest default rc=$?"
POLY_SELL_PF=3 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c4_full or c4_solve or epilogue" 2>&1 | tail -1
for i in 1 2; do
for v in 0 1 2 3; do
  POLY_SELL_PF=$v python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/bench_c4_pf$v.log 2>&1
  python - <<PY
import json
l=json.loads(open("gpurun_out/bench_c4_pf$v.log").read().strip().splitlines()[-1]); r=l["roofline"]
print("pf=$v", "step_us %.1f" % (l["ms_per_step"]*1e3), "pass_us %.1f" % (r["kernel_ms"]*1e3), "GB/s %.0f" % l["value"])
PY
done
done
POLY_SELL_PF=3 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_sell16" -s 8 -c 2 python bench.py --config c4 --no-cpu --no-e2e --steps 4 --warmup 3 > gpurun_out/ncu_pf.log 2>&1
grep -E "k_sell16|duration|dram__bytes|warps_active" gpurun_out/ncu_pf.log | head -10
