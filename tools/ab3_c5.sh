# A/B/C of libpoly variants on one config, alternating runs
# usage: bash tools/ab3_c5.sh CONFIG VARIANT...
C=$1; shift
mkdir -p gpurun_out
for i in 1 2; do
  for lib in base "$@"; do
    if [ $lib = base ]; then unset POLY_LIB_PATH; else export POLY_LIB_PATH=$PWD/build_variants/libpoly_$lib.so; fi
    python bench.py --config $C --no-cpu --no-e2e > gpurun_out/ab_${C}_${lib}_$i.log 2>&1
    python - <<PY
import json
l=json.loads(open("gpurun_out/ab_${C}_${lib}_$i.log").read().strip().splitlines()[-1]); r=l["roofline"]
print("$C $lib run $i", "step_ms %.4f" % l["ms_per_step"], "K_ms %.5f" % r["kernel_ms"], "GB/s %.0f" % l["value"], "clk", l["clocks"]["sm_mhz"] if l["clocks"] else None, l["clocks"]["reasons"] if l["clocks"] else None)
PY
  done
done
unset POLY_LIB_PATH
