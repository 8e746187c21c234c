# K1 tile sweep at C5 under the bench's (power-capped) conditions, alternating
# usage: bash tools/tune_c5.sh IDX...   (kDenseTuneF32 indices; "d" = default)
mkdir -p gpurun_out
for i in 1 2; do
  for t in d "$@"; do
    if [ $t = d ]; then unset POLY_K1_TUNE; else export POLY_K1_TUNE=$t; fi
    python bench.py --config c5 --no-cpu --no-e2e > gpurun_out/tune_c5_${t}_$i.log 2>&1
    python - <<PY
import json
l=json.loads(open("gpurun_out/tune_c5_${t}_$i.log").read().strip().splitlines()[-1]); r=l["roofline"]; d=l["config"]["tile"]
print("tile $t run $i", "step_ms %.3f" % l["ms_per_step"], "K_ms %.3f" % r["kernel_ms"], "GB/s %.0f" % l["value"], "V WPR NW RPS stages", d["V"], d["WPR"], d["NW"], d["rows_per_stage"], d["stages"], "clk", l["clocks"]["sm_mhz"])
PY
  done
done
unset POLY_K1_TUNE
