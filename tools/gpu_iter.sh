# usage: bash tools/gpu_iter.sh TAG [bench args...]
TAG=$1; shift
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py "$@" > gpurun_out/bench_$TAG.log 2>&1; tail -1 gpurun_out/bench_$TAG.log | cut -c1-2500
python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/bench_ncu_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dense_loss_grad -s 4 -c 1 \
    -o gpurun_out/prof_k1_$TAG -f python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/ncu_full_$TAG.log 2>&1
tail -2 gpurun_out/ncu_full_$TAG.log | cut -c1-300
