for v in default $VARIANTS; do
  if [ $v = default ]; then unset POLY_LIB_PATH; else export POLY_LIB_PATH=$PWD/build_variants/libpoly_$v.so; fi
  echo $v $(timeout 200 python tools/time_pb.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['matrix_free']; print(round(d['pass_ms']*1e3,1), round(d['iteration_ms']*1e3,1))")
done
