# L2 keep A/B: part of A read with evict-last so it stays in L2 across passes.
# usage: bash tools/keep_ab.sh
mkdir -p gpurun_out
run() {  # config, env
  timeout 300 env $2 python bench.py --config $1 --no-cpu --no-e2e > gpurun_out/keep_tmp.log 2>&1 || { echo "bench [$1 $2] failed"; tail -3 gpurun_out/keep_tmp.log; return; }
  python - <<PY
import json
l=json.loads(open("gpurun_out/keep_tmp.log").read().strip().splitlines()[-1]); r=l["roofline"]
print("%-4s %-28s" % ("$1", "[$2]"), "step_us %.1f" % (l["ms_per_step"]*1e3), "kernel_us %.1f" % (r["kernel_ms"]*1e3), "GB/s %.0f" % l["value"], "clk", l["clocks"]["sm_mhz"], flush=True)
PY
}
for rep in 1 2; do
  for v in "X=0" "POLY_L2_KEEP_MB=0,32" "POLY_L2_KEEP_MB=0,64" "POLY_L2_KEEP_MB=0,96" "POLY_L2_KEEP_MB=64,0" "POLY_L2_KEEP_MB=32,32" "POLY_L2_KEEP_MB=48,48" "POLY_L2_KEEP_MB=64,64"; do run c4 "$v"; done
done
for rep in 1 2; do
  for v in "X=0" "POLY_K1_KEEP_MB=32" "POLY_K1_KEEP_MB=64" "POLY_K1_KEEP_MB=96"; do run c2 "$v"; done
done
for v in "X=0" "POLY_K1_KEEP_MB=64" "POLY_K1_KEEP_MB=96"; do run c3 "$v"; done
