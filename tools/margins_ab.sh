# parity margins + C5 timing: current build vs the SFU-exp variant
mkdir -p gpurun_out
for lib in base sfu; do
  if [ $lib = base ]; then unset POLY_LIB_PATH; else export POLY_LIB_PATH=$PWD/build_variants/libpoly_$lib.so; fi
  timeout 600 python -m pytest tests/test_gpu_margins.py -q 2>&1 | tail -1
  cp gpurun_out/parity_margins.json gpurun_out/parity_margins_$lib.json
  python -c "import json; r=json.load(open('gpurun_out/parity_margins_$lib.json')); print('$lib', {k: max(v['grad_rel'] for v in d.values()) for k, d in r.items()})"
done
unset POLY_LIB_PATH
bash tools/ab3_c5.sh c5 sfu
