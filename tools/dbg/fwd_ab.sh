# forward-only in-graph cost (link kept: it resets the work counters) over variants
for v in "$@"; do
  export POLY_LIB_PATH=$PWD/build_variants/libpoly_$v.so
  for sk in none b; do
    POLY_DEV_SKIP=$sk timeout 120 python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/fab_${v}_$sk.log 2>&1
    python -c "
import json; l=json.loads(open('gpurun_out/fab_${v}_$sk.log').read().strip().splitlines()[-1]); r=l['roofline']
print('$v', '$sk', 'step %.1f' % (l['ms_per_step']*1e3), 'pass %.1f' % (r['kernel_ms']*1e3))"
  done
  timeout 120 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:k_strip_forward -s 4 -c 1 python bench.py --config c4 --no-cpu --no-e2e --steps 2 --warmup 3 2>&1 | grep -E "dram__bytes|duration"
done
