export POLY_LIB_PATH=$PWD/build_variants/libpoly_skip.so
for sk in none f l b fl lb fb; do
  POLY_DEV_SKIP=$sk timeout 120 python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/skip_$sk.log 2>&1
  python -c "
import json; l=json.loads(open('gpurun_out/skip_$sk.log').read().strip().splitlines()[-1]); r=l['roofline']
print('$sk', 'step %.1f' % (l['ms_per_step']*1e3), 'pass %.1f' % (r['kernel_ms']*1e3))"
done
