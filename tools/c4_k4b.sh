# K4b layout A/B on C4: tiled + block-synchronised (default) vs plain SELL16 columns
TAG=${1:-k4b}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py tests/test_gpu_ctproj.py -q -x -k "c4 or csr or dsell or comm or peer" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
for i in 1 2; do
for v in sync plain; do
  if [ $v = plain ]; then export POLY_K4B_PLAIN=1; else unset POLY_K4B_PLAIN; fi
  python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/bench_c4_${v}_$TAG.log 2>&1
  python - <<PY
import json
l=json.loads(open("gpurun_out/bench_c4_${v}_$TAG.log").read().strip().splitlines()[-1]); r=l["roofline"]
print("$v", "step_us %.1f" % (l["ms_per_step"]*1e3), "pass_us %.1f" % (r["kernel_ms"]*1e3), "fin_us %.1f" % (r["finalize_ms"]*1e3), "GB/s %.0f" % l["value"])
PY
done
done
unset POLY_K4B_PLAIN
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_sell16" -s 8 -c 2 python bench.py --config c4 --no-cpu --no-e2e --steps 4 --warmup 3 > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
grep -E "k_sell16|duration|dram__bytes|sectors|requests|l1tex__thr|warps_active" gpurun_out/ncu_$TAG.log | head -20
