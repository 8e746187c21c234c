# C4 e2e (poly_init included) A/B with the tiled build's phase timings on stderr
mkdir -p gpurun_out
for v in default "$@"; do
  if [ $v = default ]; then unset POLY_LIB_PATH; else export POLY_LIB_PATH=$PWD/build_variants/libpoly_$v.so; fi
  POLY_BUILD_TIMING=1 timeout 300 python bench.py --config c4 --steps 20 --no-cpu > gpurun_out/e2e_$v.log 2> gpurun_out/e2e_$v.err
  echo "== $v"; grep "tiled build" gpurun_out/e2e_$v.err | sort | uniq -c | sort -k2 | head -30
  python -c "import json;l=json.loads(open('gpurun_out/e2e_$v.log').read().strip().splitlines()[-1]);print(l['e2e']['ms_per_step'], l['ms_per_step'])"
done
