# Round-2 measurement pass: bench lines for C2/C3/C4 (default C5 is the driver's),
# a launch list of the default bench command and one ncu --set full of K1 at C5.
TAG=${1:-r02}
mkdir -p gpurun_out
for c in c2 c3 c4; do
  python bench.py --config $c > gpurun_out/bench_${c}_$TAG.log 2>&1; echo "bench $c rc=$?"
  tail -1 gpurun_out/bench_${c}_$TAG.log | cut -c1-300
done
python bench.py --no-cpu --no-e2e --steps 8 --warmup 3 > gpurun_out/plain_c5_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5_$TAG.csv \
    python bench.py --no-cpu --no-e2e --steps 8 --warmup 3 > gpurun_out/ncu_launch_c5_$TAG.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_dense_loss_grad -s 6 -c 1 \
    -o gpurun_out/prof_k1_c5_$TAG -f python bench.py --no-cpu --no-e2e --steps 4 --warmup 3 > gpurun_out/ncu_full_c5_$TAG.log 2>&1; echo "ncu full rc=$?"
