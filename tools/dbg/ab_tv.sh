python -m pytest tests/test_gpu_tv.py -q -x 2>&1 | tail -2
for v in default $VARIANTS; do
  if [ $v = default ]; then unset POLY_LIB_PATH; else export POLY_LIB_PATH=$PWD/build_variants/libpoly_$v.so; fi
  echo $v $(python tools/time_tv.py 2>&1 | tail -1)
done
