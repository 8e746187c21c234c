# matrix-free projector A/B: default build vs a variant (POLY_LIB_PATH), then the ctproj parity tests and
# per-kernel times (ncu, cold)
mkdir -p gpurun_out
for i in 1 2; do
  for lib in base "$@"; do
    if [ $lib = base ]; then unset POLY_LIB_PATH; else export POLY_LIB_PATH=$PWD/build_variants/libpoly_$lib.so; fi
    python tools/time_pb.py > gpurun_out/pb_${lib}_$i.json 2>gpurun_out/pb_${lib}_$i.err || tail -3 gpurun_out/pb_${lib}_$i.err
    python - <<PY
import json
l=json.loads(open("gpurun_out/pb_${lib}_$i.json").read().strip().splitlines()[-1])
print("$lib run $i", {k: round(v*1e3,1) for k,v in l["matrix_free"].items()}, "csr", round(l["csr"]["pass_ms"]*1e3,1))
PY
  done
done
unset POLY_LIB_PATH
timeout 600 python -m pytest tests/test_gpu_ctproj.py -m gpu -x -q 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_pb_ -s 20 -c 2 python tools/time_pb.py 2>&1 | grep -E "k_pb_|duration|inst_executed|issue_active" | sed "s/(poly::PbGeom.*//"
