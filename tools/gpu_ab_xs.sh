# K4t x-strip bulk staging: K4t/C4 tests, then A/B against HEAD's library (build_variants/libpoly_old.so)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_k4t.py -x -q > gpurun_out/k4t_tests.log 2>&1; echo "k4t tests rc=$?"; tail -2 gpurun_out/k4t_tests.log
timeout 900 python -m pytest tests -m gpu -x -q -k "c4 or C4 or csr or tiled or sell" > gpurun_out/c4_tests.log 2>&1; echo "c4 tests rc=$?"; tail -2 gpurun_out/c4_tests.log
bash tools/c4_ab.sh ${1:-xs} ${2:-old}
