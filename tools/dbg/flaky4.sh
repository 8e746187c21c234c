export POLY_L2_KEEP_MB=0,32
for lib in "$@"; do
  if [ $lib = base ]; then unset POLY_LIB_PATH; else export POLY_LIB_PATH=$PWD/build_variants/libpoly_$lib.so; fi
  echo "== $lib (keep 0,32)"; python tools/dbg/k9_flaky.py c4 0 25 1500 2>&1 | tail -1 | cut -c1-200
done
