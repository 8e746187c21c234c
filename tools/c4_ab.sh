# C4 pass A/B over libpoly variants (build_variants/libpoly_NAME.so; "default" = in-tree)
TAG=${1:-ab}; shift
mkdir -p gpurun_out
for rep in 1 2; do
for v in default "$@"; do
  if [ $v = default ]; then unset POLY_LIB_PATH; else export POLY_LIB_PATH=$PWD/build_variants/libpoly_$v.so; fi
  timeout 300 python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/bench_c4_${v}_$TAG.log 2>&1 || echo "bench $v failed"
  python - <<PY
import json
l=json.loads(open("gpurun_out/bench_c4_${v}_$TAG.log").read().strip().splitlines()[-1]); r=l["roofline"]
print("%-10s" % "$v", "step_us %.1f" % (l["ms_per_step"]*1e3), "pass_us %.1f" % (r["kernel_ms"]*1e3), "fin_us %.1f" % (r["finalize_ms"]*1e3), "GB/s %.0f" % l["value"], "clk", l["clocks"]["sm_mhz"], l["clocks"]["reasons"])
PY
done
done
unset POLY_LIB_PATH
