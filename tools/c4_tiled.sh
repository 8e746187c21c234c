# K4t (tiled CSR) vs the SELL16 pair on C4: parity tests, bench lines, ncu launch metrics.
TAG=${1:-k4t}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py tests/test_gpu_ctproj.py tests/test_gpu_fullsize.py -q -x -k "c4 or csr or dsell or comm or peer or sparse" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_$TAG.log
for v in tiled sell16; do
  if [ $v = sell16 ]; then export POLY_NO_TILED=1; else unset POLY_NO_TILED; fi
  timeout 300 python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/bench_c4_${v}_$TAG.log 2>&1; echo "bench $v rc=$?"
  python - <<PY
import json
l=json.loads(open("gpurun_out/bench_c4_${v}_$TAG.log").read().strip().splitlines()[-1]); r=l["roofline"]
print("$v", "step_us %.1f" % (l["ms_per_step"]*1e3), "pass_us %.1f" % (r["kernel_ms"]*1e3), "fin_us %.1f" % (r["finalize_ms"]*1e3), "GB/s %.0f" % l["value"], "clk", l.get("clocks"))
PY
done
unset POLY_NO_TILED
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_strip|k_tile" -s 12 -c 6 python bench.py --config c4 --no-cpu --no-e2e --steps 4 --warmup 3 > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
grep -E "k_strip|k_tile|duration|dram__bytes|warps_active|bank|inst_exec" gpurun_out/ncu_$TAG.log | head -40
