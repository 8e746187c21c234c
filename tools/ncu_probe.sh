# ncu duration + DRAM throughput of the K4t kernels for library variants
TAG=${1:-pr}; shift
for v in "$@"; do
  export POLY_LIB_PATH=$PWD/build_variants/libpoly_$v.so
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum.per_second --clock-control none -k regex:"k_strip_forward|k_tile" -s 8 -c 2 python bench.py --config c4 --no-cpu --no-e2e --steps 4 --warmup 3 > gpurun_out/ncu_probe_${v}_$TAG.log 2>&1
  echo "== $v"; grep -E "k_strip|k_tile|duration|dram__" gpurun_out/ncu_probe_${v}_$TAG.log | sed 's/(StripFwd.*//; s/(TileBwd.*//'
done
unset POLY_LIB_PATH
