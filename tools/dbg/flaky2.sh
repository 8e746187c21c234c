R=${1:-1500}
for lib in base ldonly fenceonly expconst base; do
  if [ $lib = base ]; then unset POLY_LIB_PATH; else export POLY_LIB_PATH=$PWD/build_variants/libpoly_$lib.so; fi
  echo "== $lib"; python tools/dbg/k9_flaky.py c4 0 25 $R 2>&1 | tail -1 | cut -c1-160
done
unset POLY_LIB_PATH
