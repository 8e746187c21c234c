for v in default $VARIANTS; do
  if [ $v = default ]; then unset POLY_LIB_PATH; else export POLY_LIB_PATH=$PWD/build_variants/libpoly_$v.so; fi
  echo $v; timeout 100 python tools/dbg/tv_time.py 7 100 200 256
done
timeout 60 python tools/dbg/tv_small.py 7 40 100 200 256 | grep " 50 \| 3 "
