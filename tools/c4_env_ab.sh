# C4 pass A/B over environment settings: bash tools/c4_env_ab.sh TAG "ENV1=..." "ENV2=..." (first arm: none)
TAG=${1:-env}; shift
for rep in 1 2; do
for v in "" "$@"; do
  timeout 300 env $v python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/bench_c4_env_$TAG.log 2>&1 || echo "bench [$v] failed"
  python - <<PY
import json
l=json.loads(open("gpurun_out/bench_c4_env_$TAG.log").read().strip().splitlines()[-1]); r=l["roofline"]
print("%-28s" % "[$v]", "step_us %.1f" % (l["ms_per_step"]*1e3), "pass_us %.1f" % (r["kernel_ms"]*1e3), "GB/s %.0f" % l["value"], "clk", l["clocks"]["sm_mhz"])
PY
done
done
for v in "" "$@"; do
  echo "== [$v]"
  timeout 300 env $v ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_strip|k_tile" -s 12 -c 3 python bench.py --config c4 --no-cpu --no-e2e --steps 4 --warmup 3 2>&1 | grep -E "k_strip|k_tile|duration|dram__" | sed "s/(StripFwd.*//; s/(TileBwd.*//; s/(CsrFwd.*//"
done
