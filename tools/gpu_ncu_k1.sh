set -x
python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dense_loss_grad -s 4 -c 1 \
    -o gpurun_out/prof_k1_c2 -f python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1
tail -5 gpurun_out/ncu_full.log
