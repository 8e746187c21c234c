# C4 pass A/B over libpoly variants (alternating)
mkdir -p gpurun_out
for i in 1 2; do
  for lib in base "$@"; do
    if [ $lib = base ]; then unset POLY_LIB_PATH; else export POLY_LIB_PATH=$PWD/build_variants/libpoly_$lib.so; fi
    python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/c4ab_${lib}_$i.log 2>&1
    python - <<PY
import json
l=json.loads(open("gpurun_out/c4ab_${lib}_$i.log").read().strip().splitlines()[-1]); r=l["roofline"]
print("$lib run $i", "step_us %.1f" % (l["ms_per_step"]*1e3), "pass_us %.1f" % (r["kernel_ms"]*1e3), "GB/s %.0f" % l["value"])
PY
  done
done
unset POLY_LIB_PATH
